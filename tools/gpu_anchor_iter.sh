# anchor kernel iteration: parity tests, timing probe, one ncu capture
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_dp_pins.py tests/test_gpu_full_size.py tests/test_gpu_device_es.py -x -q 2>&1 | tail -4
timeout 600 python tools/fitness_probe.py random100k 262144 ${PATHS:-anchor,anchor:16,wide} 2>&1 | tail -8
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fitness_anchor -c 1 \
  -o gpurun_out/anchor_${TAG:-new} python tools/fitness_probe.py random100k 65536 anchor > gpurun_out/ncu_anchor_${TAG:-new}.log 2>&1
tail -2 gpurun_out/ncu_anchor_${TAG:-new}.log

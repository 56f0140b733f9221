# onwalk iteration: parity tests of the wide kernels, ES fitness probe, optional full gpu suite with durations
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_dp_pins.py -x -q -m gpu 2>&1 | tail -3
timeout 600 python tools/es_fitness_probe.py random100k 1048576 2>&1 | tail -2
if [ -n "$FULL" ]; then
  timeout 3000 python -m pytest tests -m gpu -q --durations=60 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -75 gpurun_out/pytest_gpu.log
fi
if [ -n "$NCU" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fitness_onwalk -s 2 -c 1 \
    -o gpurun_out/onwalk_$NCU python tools/es_fitness_probe.py random100k 262144 > gpurun_out/ncu_onwalk_$NCU.log 2>&1
  tail -1 gpurun_out/ncu_onwalk_$NCU.log
fi

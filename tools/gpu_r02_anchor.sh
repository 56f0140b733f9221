# lockstep anchor walk iteration: parity of the wide kernels, path comparison, ES probe, ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_dp_pins.py -x -q -m gpu 2>&1 | tail -3
timeout 600 python tools/fitness_probe.py random100k 262144 ${PATHS:-onwalk,anchor:8,anchor:4,anchor:16} 2>&1 | tail -14
for p in onwalk anchor; do CB_PATH=$p timeout 600 python tools/es_fitness_probe.py random100k 1048576 2>&1 | tail -1; done
if [ -n "$NCU" ]; then
  CB_PATH=anchor timeout 900 ncu --set full --clock-control none --import-source on -k regex:fitness_anchor -s 2 -c 1 \
    -o gpurun_out/anchor_$NCU python tools/es_fitness_probe.py random100k 262144 > gpurun_out/ncu_anchor_$NCU.log 2>&1
  tail -1 gpurun_out/ncu_anchor_$NCU.log
fi

mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_dp_pins.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -2
timeout 600 python tools/fitness_probe.py random100k 262144 anchor:8,anchor:4,anchor:12 2>&1 | tail -10
CB_PATH=anchor timeout 600 python tools/es_fitness_probe.py random100k 1048576 2>&1 | tail -1
CB_PATH=anchor timeout 600 python tools/es_fitness_probe.py random100k 65536 2>&1 | tail -1
if [ -n "$NCU" ]; then
CB_PATH=anchor timeout 900 ncu --set full --clock-control none --import-source on -k regex:fitness_anchor -s 2 -c 1 \
    -o gpurun_out/anchor_$NCU python tools/es_fitness_probe.py random100k 262144 > gpurun_out/ncu_anchor_$NCU.log 2>&1
tail -1 gpurun_out/ncu_anchor_$NCU.log
fi

mkdir -p gpurun_out
CB_ANCHOR_SLOTS=1 timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_dp_pins.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -2
timeout 600 python tools/fitness_probe.py random100k 262144 anchor:8,slots 2>&1 | tail -7
for s in 0 1; do CB_ANCHOR_SLOTS=$s CB_PATH=anchor timeout 600 python tools/es_fitness_probe.py random100k 1048576 2>&1 | tail -1; done
CB_ANCHOR_SLOTS=1 CB_PATH=anchor timeout 900 ncu --set full --clock-control none --import-source on -k regex:fitness_anchor -s 2 -c 1 \
    -o gpurun_out/slots_a python tools/es_fitness_probe.py random100k 262144 > gpurun_out/ncu_slots_a.log 2>&1
tail -1 gpurun_out/ncu_slots_a.log

mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_dp_pins.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -2
timeout 600 python tools/fitness_probe.py random100k 262144 anchor:4,anchor:8 2>&1 | tail -6
for pool in 4 8; do CB_POOL=$pool CB_PATH=anchor timeout 600 python tools/es_fitness_probe.py random100k 1048576 2>&1 | tail -1; done
CB_PATH=anchor timeout 600 python tools/es_fitness_probe.py random100k 65536 2>&1 | tail -1

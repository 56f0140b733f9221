mkdir -p gpurun_out
CB_ANCHOR_GENOMES=2 timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_dp_pins.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -1
CB_ANCHOR_GENOMES=2 CB_ANCHOR_BLOCK=64 timeout 900 python -m pytest tests/test_gpu_wide.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -1
for g in 1 2; do for pool in 4 8; do for n in 65536 1048576; do CB_ANCHOR_GENOMES=$g CB_POOL=$pool CB_PATH=anchor timeout 600 python tools/es_fitness_probe.py random100k $n 2>&1 | tail -1 | sed "s/^/G $g C $pool: /"; done; done; done

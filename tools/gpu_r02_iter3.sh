mkdir -p gpurun_out
CB_ANCHOR_BLOCK=64 timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_dp_pins.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -1
for b in 128 64; do for n in 65536 262144 1048576; do CB_ANCHOR_BLOCK=$b CB_PATH=anchor timeout 600 python tools/es_fitness_probe.py random100k $n 2>&1 | tail -1 | sed "s/^/block $b: /"; done; done
timeout 300 python tools/host_profile.py random100k 2>&1 | head -40

# locate the hanging GPU test: faulthandler dumps the Python stack of a test running > 150 s
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide.py -x -q -m gpu -o faulthandler_timeout=150 -p no:cacheprovider > gpurun_out/hang.log 2>&1
tail -60 gpurun_out/hang.log
timeout 300 python tools/fitness_probe.py random100k 65536 onwalk,anchor:8 2>&1 | tail -8

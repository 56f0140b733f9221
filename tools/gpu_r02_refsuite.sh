mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_reference_suite.py tests/test_gpu_measurer.py tests/test_integration_stub.py -q -m gpu -p no:cacheprovider > gpurun_out/refsuite.log 2>&1
grep -E "^E  |FAILED|passed|failed" gpurun_out/refsuite.log | cut -c1-400 | head -60
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_dp_pins.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -2
timeout 600 python tools/fitness_probe.py random100k 262144 anchor:8,anchor:4,anchor:12,anchor:16 2>&1 | tail -13
CB_PATH=anchor timeout 600 python tools/es_fitness_probe.py random100k 1048576 2>&1 | tail -1

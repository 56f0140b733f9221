mkdir -p gpurun_out
timeout ${T:-900} python -m pytest ${TESTS:-tests/test_gpu_wide.py tests/test_dp_pins.py} -x -q -m gpu -o faulthandler_timeout=200 -p no:cacheprovider > gpurun_out/tests.log 2>&1
grep -n "Error\|error\|FAILED\|passed\|failed" gpurun_out/tests.log | head -30
tail -5 gpurun_out/tests.log

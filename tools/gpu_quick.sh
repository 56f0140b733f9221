timeout 900 python -m pytest tests/test_gpu_device_es.py tests/test_gpu_parity.py -x -q -k "device_es or breed or paths_agree or evolve" 2>&1 | tail -4
timeout 900 python bench.py 2>&1 | tail -2

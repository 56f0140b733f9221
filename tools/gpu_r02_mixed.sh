timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_gpu_parity.py tests/test_gpu_full_size.py tests/test_dp_pins.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -2
for g in 1 5; do AB_GENS=$g timeout 600 python tools/plan_ab.py nasnet_a 4194304 CB_FSM_MIXED=0,1 2>&1 | tail -2; done

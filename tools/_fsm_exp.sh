CB_FSM_STATS=1 timeout 600 python tools/host_profile.py nasnet_a 2>&1 | grep -E "fsm stats|^optimize" | cut -c1-260
nproc
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2

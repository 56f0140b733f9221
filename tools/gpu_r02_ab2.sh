AB_GENS=10 timeout 900 python tools/ab_probe.py random100k 1048576 POOL=4,6,8,12 2>&1 | tail -4
AB_GENS=10 timeout 900 python tools/ab_probe.py random100k 65536 POOL=4,8 2>&1 | tail -2
timeout 900 python tools/ab_probe.py bert_base 16777216 CB_FSM_BLOCKS=3,4 2>&1 | tail -2

timeout 900 python tools/ab_probe.py nasnet_a 4194304 CB_L2_PERSIST=0,1 2>&1 | tail -2
AB_GENS=5 timeout 900 python tools/ab_probe.py nasnet_a 4194304 CB_L2_PERSIST=0,1 2>&1 | tail -2

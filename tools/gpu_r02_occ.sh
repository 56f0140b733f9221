AB_GENS=10 timeout 900 python tools/ab_probe.py random100k 1048576 POOL=4,6,8 2>&1 | tail -3
timeout 900 python tools/ab_probe.py random100k 1048576 POOL=6,8 2>&1 | tail -2

timeout 600 python tools/ab_probe.py random100k 1048576 CB_ANCHOR_MERGE=0,1 2>&1 | tail -2
AB_GENS=10 timeout 900 python tools/ab_probe.py random100k 1048576 CB_ANCHOR_MERGE=0,1 2>&1 | tail -2
timeout 600 python tools/ab_probe.py random100k 65536 CB_ANCHOR_MERGE=0,1 CB_ANCHOR_BLOCK=64,128 2>&1 | tail -4

timeout 900 python tools/ab_probe.py random100k 65536 CB_ANCHOR_BLOCK=32,64 CB_ANCHOR_MERGE=0,1 2>&1 | tail -4
AB_GENS=10 timeout 900 python tools/ab_probe.py random100k 65536 CB_ANCHOR_BLOCK=32,64 CB_ANCHOR_MERGE=0,1 2>&1 | tail -4
timeout 900 python tools/ab_probe.py random100k 262144 CB_ANCHOR_BLOCK=32,64,128 CB_ANCHOR_MERGE=1 2>&1 | tail -3

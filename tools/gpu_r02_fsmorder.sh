for w in bert_base nasnet_a nasrnn resnet50; do AB_GENS=5 timeout 600 python tools/plan_ab.py $w 4194304 CB_FSM_ORDER=0,1 2>&1 | tail -2; done
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_gpu_parity.py tests/test_gpu_full_size.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -1

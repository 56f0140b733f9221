timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "paths_agree or fitness_matches or evolve" 2>&1 | tail -5
for w in resnet50 bert_base nasrnn nasnet_a; do timeout 300 python tools/fitness_probe.py $w 4194304 2>&1 | tail -8; done

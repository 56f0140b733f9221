timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_device_es.py -x -q -k "paths_agree or fitness_matches or evolve or device_es or breed or dp_matches" 2>&1 | tail -3
for w in resnet50 bert_base nasrnn nasnet_a; do timeout 300 python tools/fitness_probe.py $w 4194304 2>&1 | grep -E "k |frontier |unionfind" ; done

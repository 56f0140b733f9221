timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for m in bert_base nasrnn; do timeout 300 python tools/es_fitness_probe.py $m 16777216 2>&1 | tail -1; done
timeout 300 python tools/es_fitness_probe.py nasnet_a 4194304 2>&1 | tail -1

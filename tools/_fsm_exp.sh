timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python tools/fitness_probe.py nasnet_a 4194304 auto,fsm,packed_anchor 2>&1 | tail -10
timeout 300 python tools/es_fitness_probe.py nasnet_a 4194304 2>&1 | tail -1
timeout 300 python tools/es_fitness_probe.py bert_base 16777216 2>&1 | tail -1

timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for cv in 72 58 64 86; do echo "carveout $cv"; CB_FSM_CARVEOUT=$cv timeout 300 python tools/es_fitness_probe.py bert_base 16777216 2>&1 | tail -1; CB_FSM_CARVEOUT=$cv timeout 300 python tools/es_fitness_probe.py nasrnn 16777216 2>&1 | tail -1; done
timeout 600 python bench.py --no-cpu-baseline --no-configs > gpurun_out/b.json 2> gpurun_out/b.err

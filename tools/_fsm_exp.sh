timeout 300 python tools/es_fitness_probe.py bert_base 16777216 2>&1 | tail -1; timeout 300 python tools/es_fitness_probe.py nasrnn 16777216 2>&1 | tail -1; timeout 300 python tools/es_fitness_probe.py resnet50 16777216 2>&1 | tail -1
for cv in 57 43 87; do CB_FSM_CARVEOUT=$cv timeout 300 python tools/es_fitness_probe.py resnet50 16777216 2>&1 | tail -1; done
timeout 600 python bench.py --no-cpu-baseline --no-configs > gpurun_out/b.json 2> gpurun_out/b.err

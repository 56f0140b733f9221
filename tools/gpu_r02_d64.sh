# FSM walk: 16-byte vs 8-byte shared delta table (CB_FSM_D64) on ES populations, then the GPU tests
for d in 0 1; do
  echo "== CB_FSM_D64=$d"
  for m in bert_base nasrnn resnet50; do CB_FSM_D64=$d timeout 300 python tools/es_fitness_probe.py $m 16777216 2>&1 | tail -1; done
  CB_FSM_D64=$d timeout 300 python tools/es_fitness_probe.py nasnet_a 4194304 2>&1 | tail -1
done
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2

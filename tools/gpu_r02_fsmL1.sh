# FSM walk with the genome words in registers (shared words freed for L1): ES-population timings,
# ncu of one BERT-base walk, GPU tests
for m in bert_base nasrnn resnet50; do timeout 300 python tools/es_fitness_probe.py $m 16777216 2>&1 | tail -1; done
timeout 300 python tools/es_fitness_probe.py nasnet_a 4194304 2>&1 | tail -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fitness_fsm -s 2 -c 1 \
  -o gpurun_out/bert_fsm3 python tools/es_fitness_probe.py bert_base 16777216 > gpurun_out/ncu_bert_fsm3.log 2>&1; tail -1 gpurun_out/ncu_bert_fsm3.log | cut -c1-150
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2

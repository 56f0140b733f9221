# BERT-base generation: source-level ncu of the FSM walk and of the breed kernel
mkdir -p gpurun_out
ARGS="--workload bert_base --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --search-generations 2 --no-configs"
timeout 600 python bench.py $ARGS > gpurun_out/bert_plain.json 2>&1; cut -c1-300 gpurun_out/bert_plain.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fitness_fsm -s 11 -c 1 \
  -o gpurun_out/bert_fsm python bench.py $ARGS > gpurun_out/ncu_bert_fsm.log 2>&1; tail -1 gpurun_out/ncu_bert_fsm.log | cut -c1-200
timeout 900 ncu --set full --clock-control none --import-source on -k regex:breed_thread -s 7 -c 1 \
  -o gpurun_out/bert_breed python bench.py $ARGS > gpurun_out/ncu_bert_breed.log 2>&1; tail -1 gpurun_out/ncu_bert_breed.log | cut -c1-200
ls -la gpurun_out

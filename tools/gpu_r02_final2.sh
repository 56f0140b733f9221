# round-2 closing evidence (after the FSM / breed work): gpu tests, smoke, default bench + reference
# arm, BERT-base bench line, launch list of the default bench, ncu of the BERT-base FSM walk and breed
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputests.log 2>&1; tail -2 gpurun_out/gputests.log
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cut -c1-300 gpurun_out/bench.json; tail -2 gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cut -c1-200 gpurun_out/bench_ref.json
timeout 900 python bench.py --workload bert_base --no-cpu-baseline --no-configs > gpurun_out/bench_bert.json 2> gpurun_out/bench_bert.err; cut -c1-200 gpurun_out/bench_bert.json
ARGS="--steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --search-generations 3 --no-configs"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_launch_run.log 2>&1
tail -1 gpurun_out/ncu_launch_run.log | cut -c1-200
BARGS="--workload bert_base --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --search-generations 2 --no-configs"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fitness_fsm -s 11 -c 1 \
  -o gpurun_out/bert_fsm_final2 python bench.py $BARGS > gpurun_out/ncu_bert_fsm_final2.log 2>&1; tail -1 gpurun_out/ncu_bert_fsm_final2.log | cut -c1-200
timeout 900 ncu --set full --clock-control none --import-source on -k regex:breed_thread -s 7 -c 1 \
  -o gpurun_out/bert_breed_final2 python bench.py $BARGS > gpurun_out/ncu_bert_breed_final2.log 2>&1; tail -1 gpurun_out/ncu_bert_breed_final2.log | cut -c1-200
ls gpurun_out

# ncu evidence for the bench workload: launch list + full capture of the
# dominant kernel (fitness) and of the DP / matcher kernels.
mkdir -p gpurun_out
ARGS="--steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --search-generations 3 --no-configs"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_launch_run.log 2>&1
tail -2 gpurun_out/ncu_launch_run.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fitness_fsm_kernel" -s 8 -c 1 \
  -o gpurun_out/fitness_full python bench.py $ARGS > gpurun_out/ncu_full_run.log 2>&1
tail -2 gpurun_out/ncu_full_run.log
timeout 900 ncu --set full --clock-control none -k regex:"dp_narrow|match_count|match_fill|breed_thread|price_kernel" -c 6 \
  -o gpurun_out/search_full python bench.py $ARGS > gpurun_out/ncu_search_run.log 2>&1
tail -2 gpurun_out/ncu_search_run.log
ls -la gpurun_out
# the wide-program kernel (random 100k DAG, a 262 144-genome ES population after one generation)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fitness_anchor -s 2 -c 1 \
  -o gpurun_out/anchor_full python tools/es_fitness_probe.py random100k 262144 > gpurun_out/ncu_anchor_run.log 2>&1
tail -2 gpurun_out/ncu_anchor_run.log

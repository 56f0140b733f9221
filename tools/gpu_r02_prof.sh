# evidence for the bench workload: launch list of a short bench run + full capture of a timed-step fitness launch
mkdir -p gpurun_out
ARGS="--steps 2 --warmup 5 --no-cpu-baseline --e2e-steps 1 --search-generations 2 --no-configs"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_launch_run.log 2>&1
tail -1 gpurun_out/ncu_launch_run.log | cut -c1-300
# anchor launches: warm search 3, timed search 3, ES init 1 + warmup 5 -> the 13th is timed step 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fitness_anchor -s 12 -c 1 \
  -o gpurun_out/bench_fitness_full python bench.py $ARGS > gpurun_out/ncu_full_run.log 2>&1
tail -1 gpurun_out/ncu_full_run.log | cut -c1-300
timeout 600 python tools/fitness_probe.py random100k 262144 anchor:4,anchor:8 2>&1 | tail -6

# round-2 evidence: gpu tests, smoke, default bench + reference arm, launch list, ncu captures
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json; tail -2 gpurun_out/bench_ref.err
ARGS="--steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --search-generations 3 --no-configs"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_launch_run.log 2>&1
tail -2 gpurun_out/ncu_launch_run.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fitness_onwalk -s 2 -c 1 \
  -o gpurun_out/onwalk_full python tools/es_fitness_probe.py random100k 262144 > gpurun_out/ncu_onwalk_run.log 2>&1
tail -2 gpurun_out/ncu_onwalk_run.log
ls -la gpurun_out

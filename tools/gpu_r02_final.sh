# final evidence: gpu tests, smoke, default bench + reference arm, ncu capture of a timed bench generation
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cut -c1-300 gpurun_out/bench.json; tail -2 gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cut -c1-200 gpurun_out/bench_ref.json
ARGS="--steps 2 --warmup 5 --no-cpu-baseline --e2e-steps 1 --search-generations 2 --no-configs"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fitness_anchor -s 12 -c 1 \
  -o gpurun_out/bench_fitness_final python bench.py $ARGS > gpurun_out/ncu_final_run.log 2>&1
tail -1 gpurun_out/ncu_final_run.log | cut -c1-200

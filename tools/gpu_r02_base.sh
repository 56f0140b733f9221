# round-2 baseline: gpu tests, random100k bench, anchor kernel ncu capture
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py --workload random100k --population 1048576 --steps 5 --warmup 3 --no-configs --no-cpu-baseline --search-generations 10 > gpurun_out/bench100k.json 2> gpurun_out/bench100k.err; cat gpurun_out/bench100k.json; tail -3 gpurun_out/bench100k.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fitness_anchor -c 1 \
  -o gpurun_out/anchor_full_r02base python tools/fitness_probe.py random100k 262144 anchor > gpurun_out/ncu_anchor.log 2>&1
tail -2 gpurun_out/ncu_anchor.log

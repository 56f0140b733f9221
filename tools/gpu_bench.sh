# bench + ncu launch list + one full capture of the fitness kernel
mkdir -p gpurun_out
timeout 900 python bench.py 2> gpurun_out/bench.err | tee gpurun_out/bench.json
tail -5 gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
  --e2e-steps 1 --search-generations 3 > gpurun_out/ncu_launch_run.log 2>&1
tail -3 gpurun_out/ncu_launch_run.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fitness -s 8 -c 1 \
  -o gpurun_out/fitness_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  --e2e-steps 1 --search-generations 2 > gpurun_out/ncu_full_run.log 2>&1
tail -3 gpurun_out/ncu_full_run.log
ls -la gpurun_out

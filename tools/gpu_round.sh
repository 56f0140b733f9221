# full GPU check: tests, smoke, bench, ncu evidence
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2>&1; tail -1 gpurun_out/bench_ref.json
bash tools/gpu_profile.sh > gpurun_out/profile.log 2>&1; tail -3 gpurun_out/profile.log

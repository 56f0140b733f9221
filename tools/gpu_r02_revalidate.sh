# re-validation of the restored checkout: gpu tests, smoke, default bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputests.log 2>&1; tail -3 gpurun_out/gputests.log
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cut -c1-400 gpurun_out/bench.json; tail -2 gpurun_out/bench.err

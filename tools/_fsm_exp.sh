timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b.json 2> gpurun_out/b.err

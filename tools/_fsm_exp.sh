timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline --no-configs > gpurun_out/b.json 2> gpurun_out/b.err
timeout 600 ncu --set full --clock-control none --cache-control none -k regex:breed_thread -s 2 -c 1 -o gpurun_out/breed_nc3 python tools/es_fitness_probe.py bert_base 16777216 > gpurun_out/ncu_breed.log 2>&1; tail -1 gpurun_out/ncu_breed.log

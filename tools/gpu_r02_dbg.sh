mkdir -p gpurun_out
timeout 200 python tools/hang_probe.py 1:3000:64:onwalk:0 2>&1 | head -30
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_dp_pins.py -q -m gpu -o faulthandler_timeout=120 -p no:cacheprovider 2>&1 | tail -15
for p in anchor onwalk; do CB_PATH=$p timeout 600 python tools/es_fitness_probe.py random100k 1048576 2>&1 | tail -1; done
CB_PATH=anchor timeout 900 ncu --set full --clock-control none --import-source on -k regex:fitness_anchor -s 2 -c 1 \
    -o gpurun_out/anchor_c python tools/es_fitness_probe.py random100k 262144 > gpurun_out/ncu_anchor_c.log 2>&1
tail -1 gpurun_out/ncu_anchor_c.log

# timing + ncu capture of the wide (sparse warp-per-genome) fitness kernel on random100k
mkdir -p gpurun_out
timeout 600 python tools/fitness_probe.py random100k 65536 anchor,wide,unionfind 2>&1 | tail -8
timeout 600 python tools/fitness_probe.py bert_base 4194304 auto,anchor,wide 2>&1 | tail -8
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fitness_anchor -c 1 \
  -o gpurun_out/anchor_full python tools/fitness_probe.py random100k 65536 anchor > gpurun_out/ncu_wide.log 2>&1
tail -2 gpurun_out/ncu_wide.log

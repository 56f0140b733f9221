# ncu full capture of the anchor fitness kernel on random100k (65536 random genomes)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fitness_anchor -c 1 \
  -o gpurun_out/anchor_full python tools/fitness_probe.py random100k 65536 anchor > gpurun_out/ncu_anchor.log 2>&1
tail -2 gpurun_out/ncu_anchor.log

# ncu --set full of the headline anchor walk on a 262 144-genome ES population (pipe use, per-line)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fitness_anchor -s 2 -c 1 \
  -o gpurun_out/anchor_full python tools/es_fitness_probe.py random100k 262144 > gpurun_out/ncu_anchor.log 2>&1; tail -2 gpurun_out/ncu_anchor.log | cut -c1-200

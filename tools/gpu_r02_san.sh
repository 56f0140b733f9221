# compute-sanitizer on every device path (small cases) + stall profile of the search-sized anchor launch
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  for blk in 64 128; do
    CB_ANCHOR_BLOCK=$blk timeout 900 compute-sanitizer --tool $tool --print-limit 40 python tools/sanitize_probe.py > gpurun_out/san_${tool}_${blk}.log 2>&1
    echo "$tool block $blk: rc=$? $(grep -c 'ERROR SUMMARY: 0 errors' gpurun_out/san_${tool}_${blk}.log) clean summaries; $(grep 'ERROR SUMMARY' gpurun_out/san_${tool}_${blk}.log | tail -1)"
  done
done
CB_PATH=anchor timeout 900 ncu --set full --clock-control none --import-source on -k regex:fitness_anchor -s 2 -c 1 \
    -o gpurun_out/anchor_search python tools/es_fitness_probe.py random100k 65536 > gpurun_out/ncu_anchor_search.log 2>&1
tail -1 gpurun_out/ncu_anchor_search.log

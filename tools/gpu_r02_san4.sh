mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_probe.py > gpurun_out/san4_${tool}.log 2>&1
  echo "$tool rc=$?: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san4_${tool}.log | tail -1); anchor/fsm hazard lines: $(grep -cE 'fitness_anchor|fitness_fsm' gpurun_out/san4_${tool}.log)"
  grep -E "^(bert|rand|narrow|nasnet) " gpurun_out/san4_${tool}.log | cut -c1-150
done

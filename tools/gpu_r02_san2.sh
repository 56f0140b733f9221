mkdir -p gpurun_out
for blk in 64 128; do
  CB_ANCHOR_BLOCK=$blk timeout 900 compute-sanitizer --tool racecheck --print-limit 40 python tools/sanitize_probe.py > gpurun_out/san_racecheck_${blk}.log 2>&1
  echo "racecheck block $blk: $(grep 'RACECHECK SUMMARY' gpurun_out/san_racecheck_${blk}.log)"; grep -c "fitness_anchor" gpurun_out/san_racecheck_${blk}.log
done
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_dp_pins.py tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -1
for n in 65536 1048576; do CB_PATH=anchor timeout 600 python tools/es_fitness_probe.py random100k $n 2>&1 | tail -1; done
timeout 900 python bench.py --no-configs --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], 'e2e', d['e2e']['value'], 'search', d['search']['wall_s'], d['search']['es_s'])"

# default bench run (headline + five-config sweep), wall time and a summary
mkdir -p gpurun_out
s=$(date +%s)
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$? wall=$(( $(date +%s) - s ))s"
tail -3 gpurun_out/bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print({k: d[k] for k in ("value", "e2e", "roofline", "kernels_ms")})
for k, v in d.get("configs", {}).items():
    print(k, json.dumps(v))
PY

"""Dump an ncu report's details page (section / metric -> value unit) and the
top stall reasons into a JSON file under profiles/:

    python tools/ncu_details_json.py REPORT OUT.json "kernel description" "command"
"""
import csv
import json
import subprocess
import sys

rep, out, kernel, command = sys.argv[1:5]
txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
h = rows[0]
isec, iname, iunit, ival = h.index("Section Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
metrics = {f"{r[isec]} / {r[iname]}": f"{r[ival]} {r[iunit]}".strip() for r in rows[1:] if len(r) > ival}
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
names, vals = r[0], r[2]
extra = {}
for k in ("smsp__inst_executed.sum", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__t_sector_hit_rate.pct",
          "dram__bytes_read.sum", "dram__bytes_write.sum"):
    if k in names:
        extra[k] = vals[names.index(k)]
stalls = {n.replace("smsp__pcsamp_warps_issue_stalled_", ""): int(float(vals[i] or 0))
          for i, n in enumerate(names)
          if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")}
json.dump({"kernel": kernel, "command": command, "metrics": metrics, "raw": extra,
           "stall_samples_top": dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])},
          open(out, "w"), indent=1)
print(out, len(metrics), "metrics")

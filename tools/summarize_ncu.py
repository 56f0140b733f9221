"""Summarise gpurun_out/ ncu artefacts into profiles/ (run in the build
container after tools/gpu_profile.sh).  Writes:
  profiles/<tag>_launches.md          per-kernel share of the launch list
  profiles/<tag>_fitness_ncu.json     full-set metrics of the fitness kernel
  profiles/fitness_ncu_summary.json   traffic per genome (read by bench.py)
"""
import csv, json, os, subprocess, sys, collections

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = os.path.join(root, "profiles")
os.makedirs(out, exist_ok=True)

# launch list
rows = []
with open(os.path.join(root, "gpurun_out", "launches.csv")) as fh:
    lines = [l for l in fh if l.startswith('"')]
rd = csv.reader(lines)
hdr = next(rd)
ix = {h: i for i, h in enumerate(hdr)}
for r in rd:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[ix["Kernel Name"]]
    unit = r[ix["Metric Unit"]]
    v = float(r[ix["Metric Value"]].replace(",", ""))
    ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
    rows.append((name.split("(")[0], ns))
agg = collections.OrderedDict()
for n, ns in rows:
    a = agg.setdefault(n, [0, 0.0])
    a[0] += 1
    a[1] += ns
tot = sum(a[1] for a in agg.values())
with open(os.path.join(out, f"{tag}_launches.md"), "w") as fh:
    fh.write(f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none)\n\n")
    fh.write("Command: `ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 "
             "python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 "
             "--search-generations 3` (cold-cache, serialised: compare shares).\n\n")
    fh.write("| kernel | launches | total ms | share |\n|---|---:|---:|---:|\n")
    for n, (c, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        fh.write(f"| `{n}` | {c} | {ns / 1e6:.3f} | {100 * ns / tot:.1f}% |\n")
print(open(os.path.join(out, f"{tag}_launches.md")).read())

# full capture of the fitness kernel
rep = os.path.join(root, "gpurun_out", "fitness_full.ncu-rep")
if os.path.exists(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    r = list(csv.reader(raw))
    names, units, vals = r[0], r[1], r[2]
    want = ["Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
            "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct"]
    d = {}
    for w in want:
        if w in names:
            i = names.index(w)
            d[w] = {"value": vals[i], "unit": units[i]}
    stalls = {n.replace("smsp__pcsamp_warps_issue_stalled_", ""): int(float(vals[i] or 0))
              for i, n in enumerate(names)
              if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")}
    d["stall_samples"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])
    genomes = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    if genomes:
        to_b = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = float(d["dram__bytes_read.sum"]["value"]) * to_b[d["dram__bytes_read.sum"]["unit"]]
        wr = float(d["dram__bytes_write.sum"]["value"]) * to_b[d["dram__bytes_write.sum"]["unit"]]
        d["genomes_in_launch"] = genomes
        d["dram_bytes_per_genome"] = (rd + wr) / genomes
        kname = d["Kernel Name"]["value"].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        kname = kname.replace("(int)", "").replace("unsigned int", "uint32_t")
        inst = float(d["smsp__inst_executed.sum"]["value"].replace(",", ""))
        json.dump({"workload": "bert_base", "kernel": kname, "tag": tag, "genomes_in_launch": genomes,
                   "dram_bytes_per_launch_per_genome": (rd + wr) / genomes,
                   "warp_instructions_per_genome": inst / genomes,
                   "source": f"profiles/{tag}_fitness_ncu.json"},
                  open(os.path.join(out, "fitness_ncu_summary.json"), "w"), indent=1)
    json.dump(d, open(os.path.join(out, f"{tag}_fitness_ncu.json"), "w"), indent=1)
    print(json.dumps(d, indent=1))


# every full capture: one row per kernel launch (HBM roofline of each kernel)
def _rows(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    r = list(csv.reader(raw))
    if len(r) < 3:
        return []
    names, units = r[0], r[1]
    to_b = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    to_us = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
    out = []
    for vals in r[2:]:
        g = lambda k: vals[names.index(k)] if k in names else ""
        u = lambda k: units[names.index(k)] if k in names else ""
        dur = float(g("gpu__time_duration.sum").replace(",", "")) * to_us[u("gpu__time_duration.sum")]
        rd = float(g("dram__bytes_read.sum").replace(",", "")) * to_b[u("dram__bytes_read.sum")]
        wr = float(g("dram__bytes_write.sum").replace(",", "")) * to_b[u("dram__bytes_write.sum")]
        out.append((g("Kernel Name").split("(")[0], g("launch__grid_size"), dur, rd + wr,
                    g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                    g("sm__warps_active.avg.pct_of_peak_sustained_active"),
                    g("smsp__inst_executed.sum")))
    return out

peak = json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))["hbm_gbs"]
rows = []
for rep, what in (("fitness_full.ncu-rep", "bench workload (BERT-base)"),
                  ("search_full.ncu-rep", "search phase (BERT-base)"),
                  ("anchor_full.ncu-rep", "random 100k DAG, 262 144-genome ES population")):
    path = os.path.join(root, "gpurun_out", rep)
    if os.path.exists(path):
        rows += [(what,) + x for x in _rows(path)]
with open(os.path.join(out, f"{tag}_kernels.md"), "w") as fh:
    fh.write(f"# {tag}: per-kernel DRAM traffic and HBM roofline (ncu --set full, one launch each)\n\n")
    fh.write(f"Peak: {peak} GB/s (MEASURED_PEAKS.json).  ncu serialises launches and runs with cold "
             "caches; durations are for reading shares and ratios, not bench values.\n\n")
    fh.write("| workload | kernel | grid | duration us | DRAM bytes | GB/s | % of HBM peak | issue active % "
             "| warps active % | warp instructions |\n|---|---|---:|---:|---:|---:|---:|---:|---:|---:|\n")
    for what, k, grid, dur, b, iss, wa, inst in rows:
        gbs = b / (dur * 1e-6) / 1e9 if dur else 0.0
        fh.write(f"| {what} | `{k}` | {grid} | {dur:.1f} | {b:.0f} | {gbs:.2f} | {100 * gbs / peak:.4f}% "
                 f"| {iss} | {wa} | {inst} |\n")
print(open(os.path.join(out, f"{tag}_kernels.md")).read())

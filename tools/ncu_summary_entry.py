"""Add / replace a workload's entry of profiles/fitness_ncu_summary.json
(read by bench.py for roofline.traffic and issue_roofline) from one
`ncu --set full` capture of its fitness kernel:

    python tools/ncu_summary_entry.py <report.ncu-rep> <workload> <genomes in launch> <tag> <profiles json>
"""
import csv, json, os, subprocess, sys

rep, workload, genomes, tag, src = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4], sys.argv[5]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
names, units, vals = r[0], r[1], r[2]
ix = {n: i for i, n in enumerate(names)}


def val(name):
    v = float(vals[ix[name]].replace(",", ""))
    u = units[ix[name]]
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


dram = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
dur_ns = float(vals[ix["gpu__time_duration.sum"]].replace(",", "")) * {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9, "s": 1e9}[units[ix["gpu__time_duration.sum"]]]
inst = val("smsp__inst_executed.sum")
kernel = vals[ix["Kernel Name"]]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path = os.path.join(root, "profiles", "fitness_ncu_summary.json")
d = json.load(open(path)) if os.path.exists(path) else {}
d[workload] = {"kernel": kernel.split("(")[0].replace("(anonymous namespace)::", ""), "tag": tag,
               "genomes_in_launch": genomes, "dram_bytes_per_genome": dram / genomes,
               "warp_instructions_per_genome": inst / genomes, "capture_duration_s": dur_ns / 1e9,
               "capture_warp_instructions_per_s": inst / (dur_ns / 1e9), "source": src}
json.dump(d, open(path, "w"), indent=1)
print(json.dumps(d[workload], indent=1))

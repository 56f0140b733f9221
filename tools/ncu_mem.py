"""Memory counters of the first kernel in an ncu report, per unit of work
(`python tools/ncu_mem.py REPORT UNITS`)."""
import csv
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h, v = r[0], r[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
        "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum", "lts__t_sectors_srcunit_tex_op_read_evict_first_lookup_miss.sum",
        "lts__t_sectors_srcunit_tex_op_read_evict_normal_lookup_miss.sum", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]
print(v[h.index("Kernel Name")][:60])
for k in keys:
    if k in h:
        x = v[h.index(k)]
        unit = r[1][h.index(k)]
        try:
            f = float(x.replace(",", ""))
            scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(unit, None)
            per = f * scale / units if scale else f / units
            print(f"{k:70s} {x:>16s} {unit:8s} per unit {per:.2f}")
        except ValueError:
            print(k, x, unit)

"""Executed-instruction profile of an ncu report by contiguous SASS runs:
which address ranges execute how often (per `unit`, e.g. warp-steps)."""
import csv
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
for i, row in enumerate(r):
    if row and row[0] == "Address":
        hdr, start = row, i + 1
        break
ia, isrc, ix = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
rows = []
for row in r[start:]:
    try:
        rows.append((int(row[ia], 16), row[isrc].strip(), int(row[ix])))
    except (ValueError, IndexError):
        pass
base = rows[0][0]
print("per unit", sum(x[2] for x in rows) / units)
runs, cur, acc, s0 = [], None, 0.0, 0
for a, s, n in rows:
    v = round(n / units, 2)
    if cur is None or abs(v - cur) > 0.005:
        if cur is not None and acc > 0:
            runs.append((s0, a - base, cur, acc))
        cur, acc, s0 = v, 0.0, a - base
    acc += n / units
runs.append((s0, rows[-1][0] - base, cur, acc))
for s0, e0, v, acc in sorted(runs, key=lambda x: -x[3])[:top]:
    print(f"{s0:#07x}-{e0:#07x} x{v:<5} {(e0 - s0) // 16:4d} instr  {acc:6.1f}/unit")

"""Per-source-line instruction / stall-sample shares from an ncu report
(`ncu -i X --page source --csv --print-source cuda,sass`)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
for i, row in enumerate(r):
    if row and row[0] == "Line No":
        hdr, start = row, i + 1
        break
ix = hdr.index("Instructions Executed")
isamp = hdr.index("Warp Stall Sampling (All Samples)")
ith = hdr.index("Avg. Threads Executed")
rows = []
for row in r[start:]:
    if not row or not row[0].strip():
        continue
    try:
        rows.append((int(row[ix]), int(row[isamp]), row[ith], row[0], row[1][:100]))
    except (ValueError, IndexError):
        pass
tot = sum(x[0] for x in rows) or 1
ts = sum(x[1] for x in rows) or 1
print("total warp instructions", tot, "stall samples", ts)
for x in sorted(rows, reverse=True)[:top]:
    print(f"{x[0] / tot * 100:5.1f}% inst {x[1] / ts * 100:5.1f}% samp thr={x[2]:>3} L{x[3]:>4} {x[4]}")

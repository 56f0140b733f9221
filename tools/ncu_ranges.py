"""Instruction / stall-sample shares of source-line ranges from an ncu report."""
import csv, subprocess, sys
rep = sys.argv[1]
ranges = [tuple(map(int, r.split('-'))) + (r,) for r in sys.argv[2:]]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
for i, row in enumerate(r):
    if row and row[0] == "Line No":
        hdr, start = row, i + 1
        break
ix = hdr.index("Instructions Executed"); isamp = hdr.index("Warp Stall Sampling (All Samples)")
tot = [0, 0]; acc = {x[2]: [0, 0] for x in ranges}
for row in r[start:]:
    try:
        ln, n, s = int(row[0]), int(row[ix]), int(row[isamp])
    except (ValueError, IndexError):
        continue
    tot[0] += n; tot[1] += s
    for lo, hi, name in ranges:
        if lo <= ln <= hi:
            acc[name][0] += n; acc[name][1] += s
for k, v in acc.items():
    print(f"{k:12s} {100*v[0]/tot[0]:5.1f}% inst {100*v[1]/tot[1]:5.1f}% stall")

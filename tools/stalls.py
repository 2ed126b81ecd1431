"""Top warp-stall SASS lines of one kernel from `ncu --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr]
data = [r for r in rows[hdr + 1:] if len(r) == len(h) and r[0] != "Address"]
i_s = h.index("Warp Stall Sampling (All Samples)")
val = lambda r: float(r[i_s] or 0)
tot = sum(val(r) for r in data) or 1.0
for r in sorted(data, key=lambda r: -val(r))[:n]:
    print(f"{val(r) / tot * 100:5.1f}% {r[0]} {r[1][:100]}")

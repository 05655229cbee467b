"""Top stall-sampled SASS lines of one kernel from `ncu -i rep --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hi = [i for i, r in enumerate(rows) if "Address" in r and "Source" in r][0]
hdr = rows[hi]
si = hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[hi + 1:]:
    if len(r) != len(hdr):
        continue
    try:
        data.append((float(r[si] or 0), r))
    except ValueError:
        continue
tot = sum(x for x, _ in data)
for x, r in sorted(data, key=lambda t: -t[0])[:n]:
    print(f"{r[0]:>6} {100 * x / tot:5.1f}% {r[1][:100]}")
print("total samples", tot)

"""Print our kernels' durations from an ncu --csv launch list."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if "Kernel Name" in r][0]
hdr = rows[i]
for r in rows[i + 1:]:
    if len(r) < len(hdr):
        continue
    name = r[hdr.index("Kernel Name")]
    if "at::" in name:
        continue
    print(r[hdr.index("Grid Size")].ljust(14), r[hdr.index("Metric Value")].rjust(10), name[:60])

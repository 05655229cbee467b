"""Instruction mix of one kernel in an ncu report: executed warp-instructions per
opcode and the stall samples per opcode.  usage: sass_mix.py report.ncu-rep regex [top]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + pat],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
i_src, i_ex, i_st = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
ex, st = Counter(), Counter()
for r in rows[2:]:
    if len(r) <= i_ex or not r[i_ex].strip():
        continue
    toks = r[i_src].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    op = op.split(".")[0]
    ex[op] += float(r[i_ex] or 0)
    st[op] += float(r[i_st] or 0)
tot, tst = sum(ex.values()), sum(st.values()) or 1
print(f"total warp-instructions {tot:.0f}")
for op, v in ex.most_common(top):
    print(f"{op:12s} {v:12.0f} {100 * v / tot:5.1f}%   stalls {100 * st[op] / tst:5.1f}%")

"""Summarise an ncu report: key metrics per kernel and the top stall sites."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
pat = sys.argv[2] if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__inst_executed.sum", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "launch__grid_size", "launch__shared_mem_per_block_dynamic"]
for r in rows[2:]:
    if pat and pat not in r[hdr.index("Kernel Name")]:
        continue
    print({w.split(".")[0][:34]: (r[hdr.index(w)][:60] if w in hdr else None) for w in want})
if len(sys.argv) > 3:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + pat],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    h = srows[1]
    i_src, i_s = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    data, seen = [], set()
    for r in srows[2:]:
        if len(r) > i_s and r[i_s].replace(".", "").isdigit() and r[0] not in seen:
            seen.add(r[0])
            data.append(r)
    tot = sum(float(r[i_s]) for r in data) or 1
    addrs = [r[0] for r in data]
    top = sorted(data, key=lambda r: -float(r[i_s]))[:int(sys.argv[3])]
    for t in top:
        print(f"{float(t[i_s]) / tot * 100:5.1f}%  {t[0][-5:]}  {t[i_src][:90]}")
    for t in top[:3]:
        i = addrs.index(t[0])
        print("----")
        for r in data[max(0, i - 10):i + 2]:
            print(r[0][-5:], r[i_s].rjust(6), r[i_src][:90])

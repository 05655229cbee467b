"""profiles/ncu_summary.json from an `ncu --set full` report (one launch per kernel):
python tools/make_ncu_summary.py gpurun_out/prof_full.ncu-rep "<source note>" > profiles/ncu_summary.json"""
import csv
import io
import json
import subprocess
import sys

rep, note = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
        "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def col(r, name, scale=1.0):
    """value in base units (bytes, seconds) times scale"""
    try:
        i = hdr.index(name)
        return float(r[i].replace(",", "")) * UNIT.get(units[i], 1.0) * scale
    except (ValueError, IndexError):
        return None


out = {"source": note, "kernels": {}}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    short = name.split("(")[0].replace("void ", "").replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
    if short in out["kernels"]:
        continue
    rd, wr = col(r, "dram__bytes_read.sum"), col(r, "dram__bytes_write.sum")
    out["kernels"][short] = {
        "duration_us": col(r, "gpu__time_duration.sum", 1e6),
        "dram_read_MB": rd / 1e6 if rd is not None else None,
        "dram_write_MB": wr / 1e6 if wr is not None else None,
        "dram_throughput_pct": col(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "warps_active_pct": col(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "registers": col(r, "launch__registers_per_thread"),
        "grid": col(r, "launch__grid_size"),
        "l2_hit_pct": col(r, "lts__t_sector_hit_rate.pct"),
        "traffic_bytes": (rd or 0) + (wr or 0),
    }
json.dump(out, sys.stdout, indent=1)
print()

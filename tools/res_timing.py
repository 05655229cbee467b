"""Phase timeline of the resident step (GPU box): PSGD_RES_TIMING=1 stamps
globaltimer per CTA at start / end of phase 1 / end of reductions+GS / after
the grid barrier / end.  Also times the graph-replayed step (L2 flushed).
usage: python tools/res_timing.py [workload] [rank]"""
import ctypes
import os
import statistics
import sys

os.environ["PSGD_RES_TIMING"] = "1"
os.environ.setdefault("PSGD_RES_DEBUG", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1905_13727_b200 import PowerSGDEngine, _lib, catalogs  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "resnet18"
rank = int(sys.argv[2]) if len(sys.argv) > 2 else 2
eng = PowerSGDEngine(list(catalogs.get_catalog(wl).params), rank, seed=0)
eng.g[0].normal_()
buf0 = (ctypes.c_int64 * (148 * 8))()
flush = torch.empty(64 << 20, device="cuda")
for _ in range(5):
    flush.zero_()
    eng.run()
torch.cuda.synchronize()
NV = 148 * (8 + 64)
buf = (ctypes.c_int64 * NV)()
n = _lib.lib().psgd_debug_resident_times(eng.plan.handle, buf, NV)
nc = n // 72
allv = np.array(buf[:n], dtype=np.int64)
raw = allv[:nc * 8].reshape(-1, 8).astype(np.float64)
log = allv[nc * 8:].reshape(nc, 16, 4)
t = raw[:, :5]
t0 = t[:, 0].min()
t = (t - t0) / 1e3
def st(x):
    return f"min {x.min():6.2f} med {np.median(x):6.2f} max {x.max():6.2f}"

print(f"{wl} r{rank}: {t.shape[0]} CTAs (us, relative to the first CTA start)")
print("  start        ", st(t[:, 0]))
print("  phase1 dur   ", st(t[:, 1] - t[:, 0]))
print("  phase1 end   ", st(t[:, 1]))
print("  p1 end->bar  ", st(t[:, 2] - t[:, 1]))
print("  barrier out  ", st(t[:, 3]))
red_end = (raw[:, 5] - t0) / 1e3
print("  reducers end ", st(red_end[red_end > 0]))
for c in np.argsort(-(raw[:, 5] - raw[:, 3]))[:6]:
    print(f"    reducer cta {c:3d}: mat {int(raw[c, 7])}  sum {(raw[c, 6] - raw[c, 3]) / 1e3:.2f} us  mgs {(raw[c, 5] - raw[c, 6]) / 1e3:.2f} us")
print("  phase2 dur   ", st(t[:, 4] - t[:, 3]))
print("  end          ", st(t[:, 4]))
for c in list(np.argsort(-t[:, 1])[:3]) + list(np.argsort(t[:, 1])[:2]):
    segs = []
    for k in range(16):
        a, tag, p2e, _ = log[c, k]
        if a > t0 and (a - t0) / 1e3 < t[c, 1] + 0.01:
            segs.append(f"{(a - t0) / 1e3:.1f}[m{tag // 100000}c{(tag % 100000) // 10}]")
    print(f"  cta {c:3d} p1 end {t[c, 1]:.1f}; warp0 slab ends: " + " ".join(segs))
eng.capture()
ts = []
for _ in range(30):
    flush.zero_()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    eng.run()
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e) * 1e3)
print(f"  graph step median {statistics.median(ts):.2f} us")

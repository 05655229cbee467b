"""Per-CTA start/end of K1: the tail K1 leaves.  Needs the diagnostic build
    python -c "from paper_1905_13727_b200 import build as b; b.build(out='paper_1905_13727_b200/libpsgd_v_times.so', defines=['PSGD_K1_TIMES'])"
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PSGD_LIB", "paper_1905_13727_b200/libpsgd_v_times.so")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1905_13727_b200 import PowerSGDEngine, _lib, catalogs  # noqa: E402

specs = list(catalogs.get_catalog(sys.argv[1] if len(sys.argv) > 1 else "resnet18").params)
rank = int(sys.argv[2]) if len(sys.argv) > 2 else 2
eng = PowerSGDEngine(specs, rank, seed=0)
eng.g[0].normal_()
flush = torch.empty(64 * 1024 * 1024, device="cuda")
lib = _lib.lib()
fn = lib.psgd_debug_k1_times
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
out = np.zeros(3 * 1024, dtype=np.uint64)
for it in range(5):
    flush.zero_()
    eng.run()
    torch.cuda.synchronize()
    fn(out.ctypes.data, 1024)
    n = 148
    st, en, ch = out[0:3 * n:3].astype(np.int64), out[1:3 * n:3].astype(np.int64), out[2:3 * n:3]
    t0 = st.min()
    d = (en - t0) / 1e3
    s0 = (st - t0) / 1e3
    print(f"iter {it}: start spread {s0.max():.2f} us; end min {d.min():.2f} median {np.median(d):.2f} "
          f"p90 {np.percentile(d, 90):.2f} max {d.max():.2f} us; slowest CTAs {np.argsort(-d)[:5].tolist()} "
          f"chunks {[int(ch[i]) for i in np.argsort(-d)[:5]]}")

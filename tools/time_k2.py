"""Time K2 (psgd_orthogonalize) alone, L2-warm, for a catalog."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_13727_b200 import PowerSGDEngine, _lib, catalogs  # noqa: E402
from paper_1905_13727_b200.plan import ptr, stream_ptr  # noqa: E402

wl = os.environ.get("WL", "resnet18")
rank = int(os.environ.get("RANK_R", "2"))
specs = list(catalogs.stress().params if wl == "stress" else catalogs.get_catalog(wl).params)
eng = PowerSGDEngine(specs, rank, seed=0)
eng.g[0].normal_()
eng.bias_g[0].normal_()
eng.step()
lib = _lib.lib()
h, sp = eng.plan.handle, stream_ptr()
ts = []
for it in range(50):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        _lib.check(lib.psgd_orthogonalize(h, ptr(eng.P[0]), 1, ptr(eng.repl), ptr(eng.Phat), ptr(eng.bias_out),
                                          ptr(eng.status), sp), "orth")
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) / 10)
print(f"K2 {wl} r={rank}: {1e3 * statistics.median(ts):.1f} us per launch (back-to-back, L2 warm)")

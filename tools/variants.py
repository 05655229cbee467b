"""Time experiment builds of the library side by side: python tools/variants.py a.so b.so ..."""
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
flush = torch.empty(64 * 1024 * 1024, device="cuda")
for path in sys.argv[1:]:
    _lib._lib = _lib.load(path)
    eng = PowerSGDEngine(specs, rank, seed=0)
    eng.g[0].normal_()
    eng.bias_g[0].normal_()
    lib = _lib.lib()
    h, sp = eng.plan.handle, stream_ptr()
    t1, t3, tg = [], [], []
    for it in range(40):
        flush.zero_()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        eng.status.zero_()
        ev[0].record()
        _lib.check(lib.psgd_ef_p(h, ptr(eng.g[0]), ptr(eng.e[0]), ptr(eng.work[0]), ptr(eng.Q), ptr(eng.P[0]),
                                 ptr(eng.Phat), ptr(eng.repl), ptr(eng.bias_g[0]), ptr(eng.status), sp), "ef_p")
        if os.environ.get("MIDFLUSH"):
            flush.zero_()
        ev[1].record()
        _lib.check(lib.psgd_q_ef(h, ptr(eng.work[0]), ptr(eng.P[0]), 1, ptr(eng.repl), ptr(eng.Phat), ptr(eng.Q),
                                 ptr(eng.e[0]), ptr(eng.bias_out), ptr(eng.status), sp), "q_ef")
        ev[2].record()
        torch.cuda.synchronize()
        if it >= 5:
            t1.append(ev[0].elapsed_time(ev[1]))
            t3.append(ev[1].elapsed_time(ev[2]))
    eng.check()
    eng.capture()
    for it in range(40):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.run()
        b.record()
        torch.cuda.synchronize()
        if it >= 5:
            tg.append(a.elapsed_time(b))
    eng.check()
    print(f"{os.path.basename(path):28s} k1 {1e3*statistics.median(t1):7.1f}us  k3 {1e3*statistics.median(t3):7.1f}us"
          f"  graph step {1e3*statistics.median(tg):7.1f}us", flush=True)

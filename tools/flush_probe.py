"""How the L2 flush method changes the measured step (GPU box only).

Modes: none | write (256 MiB memset: leaves L2 full of DIRTY lines whose write-back
lands inside the next timed region) | write+read (memset, then read another
256 MiB buffer: L2 holds clean unrelated lines when the timed region starts).
Also times a plain 2-input streaming add of the same size for comparison.
"""
import statistics
import sys
import os

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_13727_b200 import PowerSGDEngine, catalogs  # noqa: E402

workload = sys.argv[1] if len(sys.argv) > 1 else "resnet18"
rank = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda", 0)
specs = list(catalogs.get_catalog(workload).params)
eng = PowerSGDEngine(specs, rank, seed=0, device=dev)
eng.g[0].normal_()
eng.capture()
wbuf = torch.empty(64 << 20, dtype=torch.float32, device=dev)
rbuf = torch.ones(64 << 20, dtype=torch.float32, device=dev)
sink = torch.empty(1, dtype=torch.float32, device=dev)
a = torch.randn(eng.g[0].numel(), device=dev)
b = torch.randn_like(a)
c = torch.empty_like(a)


def flush(mode):
    if mode in ("write", "write+read"):
        wbuf.zero_()
    if mode == "write+read":
        torch.sum(rbuf, out=sink)


def timeit(fn, mode, n=50):
    for _ in range(5):
        flush(mode)
        fn()
    ts = []
    for _ in range(n):
        flush(mode)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return statistics.median(ts)


for mode in ("none", "write", "write+read"):
    t_step = timeit(eng.run, mode)
    t_add = timeit(lambda: torch.add(a, b, out=c), mode)
    gbs = 3 * a.numel() * 4 / (t_add * 1e-6) / 1e9
    print(f"{workload} r{rank} flush={mode:11s} step {t_step:8.2f} us   add(3x{a.numel()*4/1e6:.1f}MB) "
          f"{t_add:7.2f} us = {gbs:7.1f} GB/s")

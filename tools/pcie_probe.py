"""PCIe probe: pinned H2D / D2H / both directions at once, at the ResNet-18 payload size,
and the host-pipelined e2e step (HostPipelinedEngine) at several group counts."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

dev = torch.device("cuda", 0)
n = 11164352 + 9728
h_in = torch.empty(n, dtype=torch.float32, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float32, pin_memory=True)
d_in = torch.empty(n, dtype=torch.float32, device=dev)
d_out = torch.empty(n, dtype=torch.float32, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    d_in.copy_(h_in, non_blocking=True)


def d2h():
    h_out.copy_(d_out, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


B = 4 * n
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = timed(fn)
    print(f"{name:5s} {ms:.3f} ms  {B / ms / 1e6:.1f} GB/s per direction")

from paper_1905_13727_b200 import catalogs  # noqa: E402
from paper_1905_13727_b200.pipeline import HostPipelinedEngine  # noqa: E402

specs = list(catalogs.get_catalog("resnet18").params)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
for groups in [int(x) for x in (sys.argv[1:] or ["4", "8", "12", "16", "24"])]:
    pipe = HostPipelinedEngine(specs, 2, groups=groups, seed=0, device=dev)
    for t in pipe.g_host + pipe.bias_host:
        t.normal_()
    for _ in range(3):
        pipe.step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pipe.step()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    pipe.check()
    ts.sort()
    print(f"e2e groups={groups:3d} ({len(pipe.groups)} actual): median {ts[len(ts) // 2]:.3f} ms  mean {sum(ts) / len(ts):.3f}")

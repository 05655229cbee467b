"""Per-group timeline of HostPipelinedEngine.step (events on the three streams)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_13727_b200 import catalogs  # noqa: E402
from paper_1905_13727_b200.pipeline import HostPipelinedEngine  # noqa: E402

dev = torch.device("cuda", 0)
specs = list(catalogs.get_catalog("resnet18").params)
groups = int(sys.argv[1]) if len(sys.argv) > 1 else 4
pipe = HostPipelinedEngine(specs, 2, groups=groups, seed=0, device=dev)
for _ in range(3):
    pipe.step()
torch.cuda.synchronize()
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
cur = torch.cuda.current_stream(dev)
t0 = E()
t0.record(cur)
for s in (pipe.s_h2d, pipe.s_cmp, pipe.s_d2h):
    s.wait_stream(cur)
ev = {}
with torch.cuda.stream(pipe.s_h2d):
    for k, e in enumerate(pipe.engines):
        a = E(); a.record(pipe.s_h2d)
        e.g[0].copy_(pipe.g_host[k], non_blocking=True)
        e.bias_g[0].copy_(pipe.bias_host[k], non_blocking=True)
        b = E(); b.record(pipe.s_h2d)
        ev[("h2d", k)] = (a, b)
with torch.cuda.stream(pipe.s_cmp):
    for k, e in enumerate(pipe.engines):
        pipe.s_cmp.wait_event(ev[("h2d", k)][1])
        a = E(); a.record(pipe.s_cmp)
        e.run(pipe.s_cmp)
        b = E(); b.record(pipe.s_cmp)
        ev[("cmp", k)] = (a, b)
with torch.cuda.stream(pipe.s_d2h):
    for k, e in enumerate(pipe.engines):
        pipe.s_d2h.wait_event(ev[("cmp", k)][1])
        a = E(); a.record(pipe.s_d2h)
        pipe.out_host[k].copy_(e.work[0], non_blocking=True)
        pipe.bias_out_host[k].copy_(e.bias_out, non_blocking=True)
        b = E(); b.record(pipe.s_d2h)
        ev[("d2h", k)] = (a, b)
cur.wait_stream(pipe.s_d2h)
t1 = E(); t1.record(cur)
torch.cuda.synchronize()
print(f"groups={groups} total {t0.elapsed_time(t1):.3f} ms")
for k in range(len(pipe.engines)):
    row = []
    for what in ("h2d", "cmp", "d2h"):
        a, b = ev[(what, k)]
        row.append(f"{what} {t0.elapsed_time(a):6.3f}-{t0.elapsed_time(b):6.3f}")
    print(f"  group {k}: {pipe.g_host[k].numel() * 4 / 1e6:6.2f} MB  " + "  ".join(row))

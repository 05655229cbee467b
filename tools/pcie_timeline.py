"""Per-group timeline of the captured HostPipelinedEngine step (timing events recorded
inside the graph on the three streams)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_13727_b200 import catalogs  # noqa: E402
from paper_1905_13727_b200.pipeline import HostPipelinedEngine  # noqa: E402

dev = torch.device("cuda", 0)
specs = list(catalogs.get_catalog("resnet18").params)
groups = int(sys.argv[1]) if len(sys.argv) > 1 else 8
pipe = HostPipelinedEngine(specs, 2, groups=groups, seed=0, device=dev, graphs=False)
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
ev = {}


def enqueue(origin):
    for s in (pipe.s_h2d, pipe.s_cmp, pipe.s_d2h):
        s.wait_stream(origin)
    t0 = E(); t0.record(origin); ev["t0"] = t0
    for s in (pipe.s_h2d, pipe.s_cmp, pipe.s_d2h):
        s.wait_event(t0)
    done_in, done_cmp = [], []
    with torch.cuda.stream(pipe.s_h2d):
        for k, e in enumerate(pipe.engines):
            a = E(); a.record(pipe.s_h2d)
            e.g[0].copy_(pipe.g_host[k], non_blocking=True)
            if e.nbias:
                e.bias_g[0].copy_(pipe.bias_host[k], non_blocking=True)
            b = E(); b.record(pipe.s_h2d)
            ev[("h2d", k)] = (a, b)
            done_in.append(b)
    with torch.cuda.stream(pipe.s_cmp):
        for k, e in enumerate(pipe.engines):
            pipe.s_cmp.wait_event(done_in[k])
            a = E(); a.record(pipe.s_cmp)
            e._enqueue(pipe.s_cmp)
            b = E(); b.record(pipe.s_cmp)
            ev[("cmp", k)] = (a, b)
            done_cmp.append(b)
    with torch.cuda.stream(pipe.s_d2h):
        for k, e in enumerate(pipe.engines):
            pipe.s_d2h.wait_event(done_cmp[k])
            a = E(); a.record(pipe.s_d2h)
            pipe.out_host[k].copy_(e.work[0], non_blocking=True)
            if e.nbias:
                pipe.bias_out_host[k].copy_(e.bias_out, non_blocking=True)
            b = E(); b.record(pipe.s_d2h)
            ev[("d2h", k)] = (a, b)
    origin.wait_stream(pipe.s_d2h)
    origin.wait_stream(pipe.s_cmp)
    t1 = E(); t1.record(origin); ev["t1"] = t1


mode = sys.argv[2] if len(sys.argv) > 2 else "graph"
if mode == "graph":
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            enqueue(s)
    torch.cuda.current_stream().wait_stream(s)
    run = g.replay
else:
    run = lambda: enqueue(torch.cuda.current_stream())  # noqa: E731
for _ in range(5):
    run()
torch.cuda.synchronize()
t0 = ev["t0"]
print(f"groups={groups} {mode} total {t0.elapsed_time(ev['t1']):.3f} ms")
for k in range(len(pipe.engines)):
    row = []
    for what in ("h2d", "cmp", "d2h"):
        a, b = ev[(what, k)]
        row.append(f"{what} {t0.elapsed_time(a):6.3f}-{t0.elapsed_time(b):6.3f}")
    print(f"  group {k}: {pipe.g_host[k].numel() * 4 / 1e6:6.2f} MB  " + "  ".join(row))

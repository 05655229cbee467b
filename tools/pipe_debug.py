"""Compare HostPipelinedEngine graph modes (debug)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_13727_b200 import catalogs  # noqa: E402
from paper_1905_13727_b200.pipeline import HostPipelinedEngine  # noqa: E402

specs = list(catalogs.RESNET18.params)
G = int(sys.argv[1]) if len(sys.argv) > 1 else 8
pa = HostPipelinedEngine(specs, 2, groups=G, seed=0, graphs="step")
pb = HostPipelinedEngine(specs, 2, groups=G, seed=0, graphs=False)
gen = torch.Generator().manual_seed(0)
for t in range(3):
    for i, s in enumerate(specs):
        x = torch.randn(s.shape, generator=gen)
        pa.grad_host_view(i).copy_(x)
        pb.grad_host_view(i).copy_(x)
    pa.step()
    pb.step()
    torch.cuda.synchronize()
    bad = []
    for i, s in enumerate(specs):
        a, b = pa.update_host_view(i), pb.update_host_view(i)
        d = (a - b).abs().max().item()
        if d > 1e-5 * max(1e-30, b.abs().max().item()):
            k, j = pa.where[i]
            ea, eb = pa.engines[k], pb.engines[k]
            dv = (ea.work[0] - eb.work[0]).abs().max().item()
            bad.append((s.name, k, d, "device diff", dv))
    print(t, "bad:", bad)

"""Minimal driver for ncu: `steps` eager PowerSGD steps of a catalog on cuda:0."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1905_13727_b200 import PowerSGDEngine, catalogs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="resnet18")
ap.add_argument("--rank", type=int, default=2)
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--workers", type=int, default=1)
ap.add_argument("--fused", action="store_true", help="heavy-ball update fused into the step")
a = ap.parse_args()
specs = list(catalogs.stress().params if a.workload == "stress" else catalogs.get_catalog(a.workload).params)
eng = PowerSGDEngine(specs, a.rank, workers=a.workers, seed=0)
for w in range(a.workers):
    eng.g[w].normal_()
    eng.bias_g[w].normal_()
if a.fused:
    eng.attach_optimizer(0.01, 0.9, fused=True, keep_update=False)
flush = torch.empty(64 * 1024 * 1024, device="cuda")
for _ in range(a.steps):
    flush.zero_()
    eng.run()
torch.cuda.synchronize()
eng.check()
print("ok")

"""Step + heavy-ball update: fused into K3's epilogue vs step() + psgd_momentum_step (GPU box)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_13727_b200 import PowerSGDEngine, catalogs  # noqa: E402

specs = list(catalogs.RESNET18.params)
flush = torch.empty(64 << 20, device="cuda")
for fused in (False, True):
    eng = PowerSGDEngine(specs, 2, seed=0)
    eng.attach_optimizer(0.01, 0.9)
    eng.g[0].normal_()
    ts = []
    for it in range(60):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        if fused:
            eng.step_with_optimizer(check=False)
        else:
            eng.run()
            eng.optimizer_step()
        b.record()
        torch.cuda.synchronize()
        if it >= 10:
            ts.append(a.elapsed_time(b) * 1e3)
    print(f"{'fused' if fused else 'separate'}: step + optimizer {statistics.median(ts):.1f} us (eager)")

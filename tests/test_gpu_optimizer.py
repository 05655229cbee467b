"""GPU: the heavy-ball update fused into the M-hat epilogue (SURVEY.md §8f row 1,
optimizer.py:131-134).  The fused path (K3 at W = 1, K5 at W > 1) must give the
same parameters and momentum buffers as the step followed by the one-pass update
kernel — bitwise, since both evaluate m = fma(mu, m, u), x -= lr (u + m) on the
same M-hat — skip failed steps, and replay identically from a CUDA graph."""

import numpy as np
import pytest
import torch

from paper_1905_13727_b200 import Communicator, ParamSpec, PowerSGDEngine, catalogs

pytestmark = pytest.mark.gpu


def _pair(specs, rank, workers=1, keep_update=True, seed=0):
    engs = []
    for fused in (False, True):
        comm = Communicator(workers) if workers > 1 else None
        e = PowerSGDEngine(specs, rank, workers=workers, comm=comm, seed=seed)
        rng = np.random.default_rng(1)
        x0 = [rng.standard_normal(s.shape).astype(np.float32) for s in specs]
        e.attach_optimizer(0.05, 0.9, params=x0, fused=fused, keep_update=keep_update)
        engs.append(e)
    return engs


def _feed(engs, specs, workers, t):
    gen = torch.Generator(device="cuda").manual_seed(100 + t)
    for w in range(workers):
        g = torch.randn(engs[0].g[w].numel(), device="cuda", generator=gen)
        b = torch.randn(engs[0].bias_g[w].numel(), device="cuda", generator=gen)
        for e in engs:
            e.g[w].copy_(g)
            e.bias_g[w].copy_(b)


@pytest.mark.parametrize("workers,keep", [(1, True), (1, False), (2, True), (3, False)])
def test_fused_update_equals_separate_update_resnet18(workers, keep):
    specs = list(catalogs.RESNET18.params)
    ref, fus = _pair(specs, 2, workers, keep_update=keep)
    assert fus.fused_in_kernel
    for t in range(3):
        _feed((ref, fus), specs, workers, t)
        ref.step()
        ref.optimizer_step()
        fus.step()
        fus.optimizer_step()  # no-op when fused
        torch.cuda.synchronize()
        assert torch.equal(ref.params, fus.params), t
        assert torch.equal(ref.mom, fus.mom), t
        assert torch.equal(ref.bias_params[:ref.nbias], fus.bias_params[:fus.nbias]), t
        assert torch.equal(ref.bias_mom[:ref.nbias], fus.bias_mom[:fus.nbias]), t
        assert torch.equal(ref.e[0], fus.e[0]) and torch.equal(ref.Q, fus.Q), t
        if keep:
            assert torch.equal(ref.work[0], fus.work[0]), t


def test_fused_update_falls_back_on_plans_k3_cannot_fuse():
    """Tall matrices at W = 1 (K4 writes M-hat): the update runs as the one-pass kernel
    appended to the step; results equal the unfused step + optimizer_step."""
    specs = [ParamSpec("tall", (2600, 650)), ParamSpec("b", (32,)), ParamSpec("w", (64, 576))]
    ref, fus = _pair(specs, 4)
    assert not fus.fused_in_kernel
    for t in range(2):
        _feed((ref, fus), specs, 1, t)
        ref.step()
        ref.optimizer_step()
        fus.step()
        torch.cuda.synchronize()
        assert torch.equal(ref.params, fus.params) and torch.equal(ref.mom, fus.mom), t


def test_fused_update_skips_a_failed_step_and_replays_from_a_graph():
    specs = list(catalogs.RESNET18.params)
    ref, fus = _pair(specs, 2)
    fus.capture()
    for t in range(2):
        _feed((ref, fus), specs, 1, t)
        ref.step()
        ref.optimizer_step()
        fus.run()
    torch.cuda.synchronize()
    assert torch.equal(ref.params, fus.params) and torch.equal(ref.mom, fus.mom)
    x0, m0 = fus.params.clone(), fus.mom.clone()
    bx0 = fus.bias_params.clone()
    fus.g[0][12345] = float("nan")
    fus.run()
    torch.cuda.synchronize()
    with pytest.raises(Exception):
        fus.check()
    assert torch.equal(fus.params, x0) and torch.equal(fus.mom, m0) and torch.equal(fus.bias_params, bx0)

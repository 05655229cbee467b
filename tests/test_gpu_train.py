"""GPU: end-to-end training through the drop-in.

The reference's own known-answer training run, GOLDEN_TRAIN_CSV
(pkg/tests/test_cli.py:10-17: powersgd rank 2, 2 workers, seed 1, least
squares 24 x 32, lr 0.01, momentum 0.9), replayed with the compression step
AND the heavy-ball update (optimizer.py:131-134) on the B200 path: gradients
come from the desk problem on the host (train.py:78-139 computes them
outside the optimizer too), everything else runs on the device.  Losses match
the reference's float64 values to fp32 tolerance; bits and decode_ops exactly.
"""

import numpy as np
import pytest
import torch

from oracle import powersgd as O
from paper_1905_13727_b200 import Communicator, ParamSpec, PowerSGDEngine

from test_oracle import GOLDEN_TRAIN

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fused", [False, True])
def test_golden_train_csv_replayed_on_gpu(fused):
    """fused=True: the heavy-ball update runs inside K5 (psgd_decompress_sgd)."""
    seed, world, rank, lr, mom = 1, 2, 2, 0.01, 0.9
    prob = O.LeastSquares(seed)
    specs = [ParamSpec(s.name, s.shape) for s in prob.specs]
    comm = Communicator(world)
    eng = PowerSGDEngine(specs, rank, workers=world, comm=comm, seed=seed)
    eng.attach_optimizer(lr, mom, params=prob.init_params(), fused=fused)
    assert eng.fused_in_kernel == fused
    rows = [(0, prob.loss(prob.init_params()), 0, 0)]
    for t in range(3):
        params = [eng.param_view(i).double().cpu().numpy() for i in range(len(specs))]
        for w in range(world):
            for i, g in enumerate(prob.worker_gradients(params, w, world)):
                eng.grad_view(i, w).copy_(torch.from_numpy(g.astype(np.float32)))
        eng.step()
        eng.optimizer_step()
        params = [eng.param_view(i).double().cpu().numpy() for i in range(len(specs))]
        rows.append((t + 1, prob.loss(params), comm.stats.bits_allreduced, comm.stats.decode_ops))
    for got, want in zip(rows, GOLDEN_TRAIN):
        assert got[0] == want[0] and got[2] == want[2] and got[3] == want[3], (got, want)
        assert abs(got[1] - want[1]) <= 1e-5 * abs(want[1]), (got, want)


@pytest.mark.parametrize("fused", [False, True])
def test_momentum_kernel_matches_reference_update(fused):
    """fused=True: the update runs in K3's epilogue (psgd_step_single_sgd), including
    the scalar (m % 4 != 0) slab path of (10, 27)."""
    specs = [ParamSpec("w", (64, 576)), ParamSpec("b", (64,)), ParamSpec("v", (10, 27))]
    eng = PowerSGDEngine(specs, 2)
    rng = np.random.default_rng(0)
    x0 = [rng.standard_normal(s.shape) for s in specs]
    eng.attach_optimizer(0.05, 0.9, params=x0, fused=fused)
    assert eng.fused_in_kernel == fused
    xs = [a.copy() for a in x0]
    bufs = [np.zeros(s.shape) for s in specs]
    for _ in range(3):
        grads = [rng.standard_normal(s.shape).astype(np.float32) for s in specs]
        for i, g in enumerate(grads):
            eng.grad_view(i).copy_(torch.from_numpy(g))
        eng.step()
        eng.optimizer_step()
        ups = [eng.update_view(i).double().cpu().numpy() for i in range(len(specs))]
        O.momentum_update(xs, bufs, ups, 0.05, 0.9)
        for i in range(len(specs)):
            np.testing.assert_allclose(eng.param_view(i).cpu().numpy(), xs[i], rtol=1e-5, atol=1e-6)
            np.testing.assert_allclose(eng.momentum_view(i).cpu().numpy(), bufs[i], rtol=1e-5, atol=1e-6)

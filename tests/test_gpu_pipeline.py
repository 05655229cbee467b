"""GPU: HostPipelinedEngine (host gradients in, host update out, transfers
overlapped with compression) equals the single-engine step and the oracle."""

import numpy as np
import pytest
import torch

from oracle import powersgd as O
from paper_1905_13727_b200 import PowerSGDEngine, catalogs
from paper_1905_13727_b200.pipeline import HostPipelinedEngine, split_groups

pytestmark = pytest.mark.gpu


def test_groups_cover_the_catalog_in_order():
    specs = list(catalogs.RESNET18.params)
    gs = split_groups(specs, 4)
    assert [i for g in gs for i in g] == list(range(len(specs))) and len(gs) == 4


@pytest.mark.parametrize("groups,graphs", [(8, "step"), (4, "engine"), (5, False)])
def test_pipelined_host_step_matches_engine_and_oracle(groups, graphs):
    specs = list(catalogs.RESNET18.params)
    pipe = HostPipelinedEngine(specs, 2, groups=groups, seed=0, graphs=graphs)
    ref = PowerSGDEngine(specs, 2, seed=0)
    ospecs = [O.ParamSpec(s.name, s.shape) for s in specs]
    comp, comm, workers = O.PowerSGD(2), O.Communicator(1), [O.WorkerState(0)]
    for t in range(2):
        grads = [O.derive_rng(0, "grad", t, 0, i).standard_normal(s.shape).astype(np.float32)
                 for i, s in enumerate(specs)]
        for i, g in enumerate(grads):
            pipe.grad_host_view(i).copy_(torch.from_numpy(g))
            ref.grad_view(i).copy_(torch.from_numpy(g))
        pipe.step()
        ref.step()
        torch.cuda.synchronize()
        pipe.check()
        updates, _ = O.ef_step(workers, [grads], ospecs, comp, comm, 0, t)
        for i, s in enumerate(specs):
            got = pipe.update_host_view(i).double().numpy()
            want = ref.update_view(i).double().cpu().numpy()
            assert np.linalg.norm(got - want) <= 1e-6 * max(np.linalg.norm(want), 1e-30), (t, s.name)
            err = np.linalg.norm(got.reshape(updates[i].shape) - updates[i]) / max(np.linalg.norm(updates[i]), 1e-30)
            assert err <= 1e-4, (t, s.name, err)

"""GPU: the DDP communication hook.

Two DDP ranks share cuda:0 over gloo.  After backward, every parameter's
.grad must equal the reference's aggregated update for the two ranks' raw
gradients (optimizer.py:110-129 via the CPU oracle at W = 2): M-hat for
matrices, the mean for biases; two steps, so error feedback and the warm
start carry over between calls.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import powersgd as O

pytestmark = pytest.mark.gpu
WORLD = 2


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def make_model():
    torch.manual_seed(0)
    return torch.nn.Sequential(torch.nn.Conv2d(3, 8, 3), torch.nn.ReLU(), torch.nn.Flatten(),
                               torch.nn.Linear(8 * 6 * 6, 24), torch.nn.ReLU(), torch.nn.Linear(24, 5))


def batch(rank, step):
    g = torch.Generator().manual_seed(100 * step + rank)
    return torch.randn(4, 3, 8, 8, generator=g), torch.randn(4, 5, generator=g)


def worker(rank, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from paper_1905_13727_b200.ddp import PowerSGDState, powersgd_hook
    dev = torch.device("cuda", 0)
    model = make_model().to(dev)
    ref = make_model().to(dev)  # same init: raw gradients of both ranks for the oracle
    ddp = torch.nn.parallel.DistributedDataParallel(model, bucket_cap_mb=0.002)
    state = PowerSGDState(model, rank=2, seed=0)
    ddp.register_comm_hook(state, powersgd_hook)
    names = [n for n, _ in model.named_parameters()]
    ospecs = [O.ParamSpec(n, tuple(p.shape)) for n, p in model.named_parameters()]
    comp, comm = O.PowerSGD(2), O.Communicator(WORLD)
    workers = [O.WorkerState(w) for w in range(WORLD)]
    worst = 0.0
    for step in range(2):
        x, y = batch(rank, step)
        ddp.zero_grad(set_to_none=True)
        torch.nn.functional.mse_loss(ddp(x.to(dev)), y.to(dev)).backward()
        torch.cuda.synchronize()
        grads = []
        for w in range(WORLD):
            xw, yw = batch(w, step)
            ref.zero_grad(set_to_none=True)
            torch.nn.functional.mse_loss(ref(xw.to(dev)), yw.to(dev)).backward()
            grads.append([p.grad.detach().cpu().numpy().astype(np.float32) for p in ref.parameters()])
        updates, _ = O.ef_step(workers, grads, ospecs, comp, comm, 0, step)
        for i, p in enumerate(model.parameters()):
            got = p.grad.detach().double().cpu().numpy()
            den = max(np.linalg.norm(updates[i]), 1e-30)
            worst = max(worst, float(np.linalg.norm(got - updates[i]) / den))
    np.save(os.path.join(out, f"rank{rank}.npy"), np.array([worst, len(state.engines)]))
    del names
    dist.barrier()
    dist.destroy_process_group()


def test_ddp_hook_matches_reference_aggregate(tmp_path):
    mp.spawn(worker, args=(free_port(), str(tmp_path)), nprocs=WORLD, join=True)
    for r in range(WORLD):
        worst, nb = np.load(tmp_path / f"rank{r}.npy")
        assert worst <= 1e-4, (r, worst)
        assert nb >= 2  # several buckets: compression overlapped backward bucket by bucket

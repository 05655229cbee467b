"""GPU: the one-worker-per-process exchange path on a real device.

Two processes share cuda:0 and exchange through gloo (CUDA tensors), so the
exact multi-GPU kernel sequence runs at W = 2: K1 -> all_reduce(P | bias |
flags) -> K2/K3 (÷W fused) -> all_reduce(q) -> K5.  Only the transport differs
from the NCCL path (NCCL refuses two ranks on one GPU; this run has one GPU).
Each rank checks P-hat, Q-bar, M-hat and its own e_w against the CPU oracle
running the reference's W = 2 step (optimizer.py:110-129) on the same inputs.
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
TOL = 1e-4


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def worker(rank, port, out_dir, catalog, rank_r, steps):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from paper_1905_13727_b200 import DistributedCommunicator, ParamSpec, PowerSGDEngine, catalogs
    if catalog == "odd":
        specs = [ParamSpec("a", (8, 6)), ParamSpec("bias", (10,)), ParamSpec("c", (16, 3, 2, 2)),
                 ParamSpec("d", (700, 33)), ParamSpec("e", (5, 1)), ParamSpec("bias2", (3,))]
    else:
        specs = list(catalogs.get_catalog(catalog).params)
    comm = DistributedCommunicator()
    eng = PowerSGDEngine(specs, rank_r, comm=comm, seed=0)
    ospecs = [O.ParamSpec(s.name, s.shape) for s in specs]
    comp, ocomm = O.PowerSGD(rank_r), O.Communicator(WORLD)
    workers = [O.WorkerState(w) for w in range(WORLD)]
    errs = {"p": 0.0, "q": 0.0, "mhat": 0.0, "e": 0.0, "bias": 0.0}
    for t in range(steps):
        grads = [[O.derive_rng(0, "grad", t, w, i).standard_normal(s.shape).astype(np.float32)
                  for i, s in enumerate(specs)] for w in range(WORLD)]
        for i in range(len(specs)):
            eng.grad_view(i).copy_(torch.from_numpy(grads[rank][i]))
        eng.step()
        updates, payloads = O.ef_step(workers, grads, ospecs, comp, ocomm, 0, t)
        for i, s in enumerate(specs):
            if s.is_bias:
                errs["bias"] = max(errs["bias"], rel(eng.update_view(i).cpu(), updates[i]))
                continue
            errs["p"] = max(errs["p"], rel(eng.p_view(i).cpu(), payloads[i].p))
            errs["q"] = max(errs["q"], rel(eng.q_view(i).cpu(), payloads[i].q))
            errs["mhat"] = max(errs["mhat"], rel(eng.update_view(i).cpu(), updates[i]))
            n, m = s.matrix_shape
            e_ref = workers[rank].error[i]
            den = np.linalg.norm(grads[rank][i].reshape(n, m).astype(np.float64)) \
                if min(n, m, rank_r) == min(n, m) else np.linalg.norm(e_ref)
            errs["e"] = max(errs["e"], float(np.linalg.norm(eng.error_view(i).cpu().numpy() - e_ref) / den))
    stats = np.array([eng.stats.bits_allreduced, eng.stats.compress_flops, eng.stats.decode_ops])
    ostats = np.array([ocomm.stats.bits_allreduced, ocomm.stats.compress_flops, ocomm.stats.decode_ops])
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), errs=np.array([errs[k] for k in sorted(errs)]),
             stats=stats, ostats=ostats)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("catalog,rank_r,steps", [("resnet18", 2, 2), ("odd", 3, 2), ("lstm", 4, 1)])
def test_exchange_path_matches_oracle_at_w2(tmp_path, catalog, rank_r, steps):
    mp.spawn(worker, args=(free_port(), str(tmp_path), catalog, rank_r, steps), nprocs=WORLD, join=True)
    for r in range(WORLD):
        z = np.load(tmp_path / f"rank{r}.npz")
        assert float(z["errs"].max()) <= TOL, (r, z["errs"])
        assert np.array_equal(z["stats"], z["ostats"]), (z["stats"], z["ostats"])

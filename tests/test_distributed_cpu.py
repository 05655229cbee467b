"""The one-worker-per-GPU exchange, host side, on CPU with gloo (world size 2).

Covers what the NCCL path does between the kernels: the packed AR1 payload
(P ⊕ bias ⊕ non-finite flags) and AR2 payload (q) summed across workers and
divided by W reproduce the reference's tree mean (comm.py:84-98), CommStats
charging equals the reference's optimizer.step charging, a non-finite flag on
one rank reaches every rank, and the first non-finite site is named exactly as
optimizer.py:72-76 scans (worker-major)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import powersgd as O

WORLD = 2


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


SPECS = [O.ParamSpec("a", (8, 6)), O.ParamSpec("bias", (10,)), O.ParamSpec("c", (16, 12)),
         O.ParamSpec("d", (5, 3, 2))]
RANK_R = 2


def worker(rank, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from paper_1905_13727_b200.comm import DistributedCommunicator
    from paper_1905_13727_b200.distributed import first_nonfinite_site, reduce_packed_, step_charges
    comm = DistributedCommunicator()
    res = {}
    # --- AR1: pack [P of every matrix | bias | flags], sum, / W  vs the oracle tree mean
    mats = [s for s in SPECS if not s.is_bias]
    pw = [O.derive_rng(3, "p", rank, i).standard_normal((s.matrix_shape[0], RANK_R)).astype(np.float32)
          for i, s in enumerate(mats)]
    bias = O.derive_rng(3, "bias", rank).standard_normal(10).astype(np.float32)
    flags = np.zeros(4, np.float32)
    if rank == 1:
        flags[2] = 1.0  # this rank saw a non-finite gradient
    buf = torch.from_numpy(np.concatenate([p.ravel() for p in pw] + [bias, flags]))
    reduce_packed_(buf, comm)
    res["p_mean"] = (buf / WORLD).numpy()
    # --- AR2 on q
    q = torch.from_numpy(O.derive_rng(3, "q", rank).standard_normal(40).astype(np.float32))
    reduce_packed_(q, comm)
    res["q_mean"] = (q / WORLD).numpy()
    # --- accounting
    res["charges"] = np.array(step_charges([(s.matrix_shape[0], s.matrix_shape[1],
                                             min(*s.matrix_shape, RANK_R)) for s in mats], 10, WORLD))
    # --- first non-finite site: rank 1 has a bad param 2, rank 0 a clean step
    site = first_nonfinite_site(2 if rank == 1 else None, comm, len(SPECS))
    res["site"] = np.array(site)
    site_none = first_nonfinite_site(None, comm, len(SPECS))
    res["site_none"] = np.array(-1 if site_none is None else 0)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    dist.barrier()
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def results(tmp_path_factory):
    out = tmp_path_factory.mktemp("dist")
    mp.spawn(worker, args=(free_port(), str(out)), nprocs=WORLD, join=True)
    return [np.load(out / f"rank{r}.npz") for r in range(WORLD)]


def test_packed_p_allreduce_is_the_reference_tree_mean(results):
    mats = [s for s in SPECS if not s.is_bias]
    want_parts = []
    for i, s in enumerate(mats):
        per = [O.derive_rng(3, "p", r, i).standard_normal((s.matrix_shape[0], RANK_R)).astype(np.float32)
               .astype(np.float64) for r in range(WORLD)]
        want_parts.append(O.Communicator(WORLD).all_reduce_mean(per).ravel())
    bias = [O.derive_rng(3, "bias", r).standard_normal(10).astype(np.float32).astype(np.float64)
            for r in range(WORLD)]
    want = np.concatenate(want_parts + [O.Communicator(WORLD).all_reduce_mean(bias)])
    for res in results:  # identical on every rank, equal to the tree mean to fp32 rounding
        got = res["p_mean"][:want.size]
        np.testing.assert_allclose(got, want, rtol=1e-6, atol=1e-7)
        assert np.array_equal(res["p_mean"], results[0]["p_mean"])


def test_nonfinite_flag_reaches_every_rank(results):
    for res in results:
        flags = res["p_mean"][-4:]
        assert flags[2] > 0 and flags[0] == 0


def test_q_allreduce(results):
    per = [O.derive_rng(3, "q", r).standard_normal(40).astype(np.float32).astype(np.float64) for r in range(WORLD)]
    want = O.Communicator(WORLD).all_reduce_mean(per)
    for res in results:
        np.testing.assert_allclose(res["q_mean"], want, rtol=1e-6, atol=1e-7)


def test_charges_match_reference_step(results):
    comm = O.Communicator(WORLD)
    workers = [O.WorkerState(w) for w in range(WORLD)]
    grads = [[O.derive_rng(5, "g", w, i).standard_normal(s.shape) for i, s in enumerate(SPECS)]
             for w in range(WORLD)]
    O.ef_step(workers, grads, SPECS, O.PowerSGD(RANK_R), comm, 0, 0)
    want = (comm.stats.bits_allreduced, comm.stats.compress_flops, comm.stats.decode_ops)
    for res in results:
        assert tuple(int(x) for x in res["charges"]) == want


def test_first_nonfinite_site_is_worker_major(results):
    for res in results:
        assert tuple(int(x) for x in res["site"]) == (2, 1)
        assert int(res["site_none"]) == -1

"""The reference's own PowerSGD / orthogonalize tests, re-run through the B200
drop-in API (pkg/tests/test_compressors.py:93-183, test_linalg.py:43-97,
test_optimizer.py:94-110).  Tolerances that the reference states for float64
(1e-12) are restated for the fp32 path and say so."""

import os

import numpy as np
import pytest
import torch

from oracle import powersgd as O
from paper_1905_13727_b200 import (Communicator, CompressionContext, ContractViolation, decompress,
                                   make_compressor, orthogonalize)
from paper_1905_13727_b200.seeding import derive_rng

pytestmark = pytest.mark.gpu

FP32 = 2e-6  # fp32 replacement for the reference's 1e-12 orthonormality bound


def ctx_at(step=0, param=0, seed=123):
    return CompressionContext(shared_seed=seed, param_index=param, step=step)


def worker_mats(world, n=8, m=6, seed=900):
    rng = derive_rng(seed, "worker_mats")
    return [rng.standard_normal((n, m)) for _ in range(world)]


def test_rank_clamps_to_matrix_dims():
    comp = make_compressor("powersgd", rank=5)
    assert comp.effective_rank(3, 7) == 3
    payload = comp.compress(derive_rng(902, "clamp").standard_normal((3, 7)), ctx_at())
    assert payload.p.shape == (3, 3) and payload.q.shape == (7, 3)


def test_payload_shapes_and_orthonormal_p():
    rt = make_compressor("powersgd", rank=2).round_trip(worker_mats(3), ctx_at(), Communicator(3))
    assert rt.payload.p.shape == (8, 2) and rt.payload.q.shape == (6, 2)
    assert np.max(np.abs(rt.payload.p.T @ rt.payload.p - np.eye(2))) <= FP32


def test_round_trip_matches_oracle_round_trip():
    for world in (1, 2, 3, 4):
        mats = worker_mats(world, n=33, m=20)
        ours = make_compressor("powersgd", rank=3).round_trip(mats, ctx_at(param=7), Communicator(world))
        mats32 = [m.astype(np.float32).astype(np.float64) for m in mats]
        ref = O.PowerSGD(3).round_trip(mats32, O.CompressionContext(123, 7, 0), O.Communicator(world))
        for a, b in [(ours.aggregated, ref.aggregated), (ours.payload.p, ref.payload.p),
                     (ours.payload.q, ref.payload.q)] + list(zip(ours.locals, ref.locals)):
            assert np.linalg.norm(a - b) <= 1e-5 * np.linalg.norm(b)


def test_warm_start_converges_on_a_fixed_matrix():
    rng = derive_rng(903, "warm")
    mat = rng.standard_normal((16, 12))
    comp = make_compressor("powersgd", rank=2)
    u, s, vt = np.linalg.svd(mat)
    target = float(np.sqrt(np.sum(s[2:] ** 2)))
    errs = []
    for step in range(40):
        payload = comp.compress(mat, ctx_at(step=step))
        errs.append(float(np.linalg.norm(mat - decompress(payload))))
    assert errs[-1] <= target * (1 + 1e-5)
    assert errs[0] > errs[-1]


def test_compress_of_compressed_is_identity():
    mat = derive_rng(904, "proj").standard_normal((10, 7))
    y1 = decompress(make_compressor("powersgd", rank=2).compress(mat, ctx_at()))
    y2 = decompress(make_compressor("powersgd", rank=2).compress(y1, ctx_at()))
    assert np.max(np.abs(y2 - y1)) <= 1e-5 * np.max(np.abs(y1))


def test_aggregate_matches_mean_input():
    mats = worker_mats(4, n=12, m=10, seed=905)
    mean = O.tree_reduce(mats, lambda a, b: a + b) / 4
    rt = make_compressor("powersgd", rank=2).round_trip(mats, ctx_at(), Communicator(4))
    alone = decompress(make_compressor("powersgd", rank=2).compress(mean, ctx_at()))
    assert np.max(np.abs(rt.aggregated - alone)) <= 1e-5 * np.max(np.abs(alone))


def test_locals_are_projections_of_own_matrix():
    mats = worker_mats(2)
    rt = make_compressor("powersgd", rank=2).round_trip(mats, ctx_at(), Communicator(2))
    p = rt.payload.p
    for mat, local in zip(mats, rt.locals):
        assert np.max(np.abs(local - p @ (mat.T @ p).T)) <= 1e-5


def test_warm_start_is_per_parameter():
    comp = make_compressor("powersgd", rank=1)
    a = derive_rng(906, "a").standard_normal((5, 4))
    comp.compress(a, ctx_at(param=0))
    comp.compress(a, ctx_at(param=3))
    assert set(comp.q_memory) == {0, 3}


def test_accounting_matches_reference():
    mats = worker_mats(3, n=6, m=5)
    comm = Communicator(3)
    comp = make_compressor("powersgd", rank=2)
    comp.round_trip(mats, ctx_at(), comm)
    ref_comm = O.Communicator(3)
    O.PowerSGD(2).round_trip(mats, O.CompressionContext(123), ref_comm)
    assert (comm.stats.bits_allreduced, comm.stats.decode_ops, comm.stats.compress_flops) == \
        (ref_comm.stats.bits_allreduced, ref_comm.stats.decode_ops, ref_comm.stats.compress_flops)


def test_world_size_mismatch_and_nonfinite():
    comp = make_compressor("powersgd", rank=2)
    with pytest.raises(ValueError):
        comp.round_trip(worker_mats(2), ctx_at(), Communicator(3))
    bad = worker_mats(1)[0]
    bad[2, 3] = np.nan
    with pytest.raises(ContractViolation):
        comp.round_trip([bad], ctx_at(), Communicator(1))


def test_tensor_mode_defers_errors_to_check_and_numpy_q_memory():
    """CUDA-tensor calls do not synchronise: a non-finite input is raised by check();
    numpy calls keep q_memory as float64 numpy (compressors.py:357, :373), and repeated
    calls reuse the cached workspace and the device mirror of Q (same results as a
    fresh compressor fed the same q_memory)."""
    comp = make_compressor("powersgd", rank=2)
    bad = torch.randn(30, 20, device="cuda")
    bad[1, 1] = float("nan")
    comp.round_trip([bad], ctx_at(), Communicator(1))  # no raise here
    with pytest.raises(ContractViolation):
        comp.check()
    comp.check()  # cleared
    mats = worker_mats(1, n=30, m=20)
    a1 = comp.round_trip(mats, ctx_at(param=5), Communicator(1))
    assert isinstance(comp.q_memory[5], np.ndarray) and comp.q_memory[5].dtype == np.float64
    a2 = comp.round_trip(mats, ctx_at(param=5, step=1), Communicator(1))
    comp2 = make_compressor("powersgd", rank=2)
    comp2.q_memory[5] = a1.payload.q.copy()
    b2 = comp2.round_trip(mats, ctx_at(param=5, step=1), Communicator(1))
    np.testing.assert_array_equal(a2.aggregated, b2.aggregated)
    np.testing.assert_array_equal(a2.payload.q, b2.payload.q)


def test_torch_tensors_in_and_out():
    mats = [torch.randn(40, 24, device="cuda") for _ in range(2)]
    rt = make_compressor("powersgd", rank=2).round_trip(mats, ctx_at(), Communicator(2))
    assert isinstance(rt.aggregated, torch.Tensor) and rt.aggregated.is_cuda
    assert rt.aggregated.dtype == torch.float32 and rt.payload.p.shape == (40, 2)


@pytest.mark.parametrize("key", ["rand_12x1", "rand_12x2", "rand_64x5", "rand_513x8", "dup_zero_9x3",
                                 "opposite_7x2", "ones_6x2", "zero_5x2", "square_4x4"])
def test_orthogonalize_matches_reference_fixture(golden_dir, key):
    z = np.load(os.path.join(golden_dir, "orthogonalize.npz"))
    p = z[f"in_{key}"].astype(np.float32)
    got = orthogonalize(p)
    r = p.shape[1]
    assert np.max(np.abs(got.T @ got - np.eye(r))) <= FP32
    want = O.orthogonalize(p.astype(np.float64))  # same fp32 input, float64 oracle
    assert np.linalg.norm(got - want) <= 1e-5 * np.linalg.norm(want), key
    # the reference's own output on its float64 input (equal to fp32 rounding)
    assert np.linalg.norm(got - z[f"out_{key}"]) <= 1e-4 * np.linalg.norm(z[f"out_{key}"]), key


def test_orthogonalize_rejects_bad_input():
    with pytest.raises(ContractViolation):
        orthogonalize(np.zeros((2, 3)))
    with pytest.raises(ContractViolation):
        orthogonalize(np.array([[1.0, np.inf], [0.0, 1.0]]))


def test_degenerate_opposite_workers_give_zero_update():
    # SPEC.md worked example: M1 = -M2 -> P = 0 -> replacement frame, Q = 0, M-hat = 0
    m = np.arange(12.0).reshape(3, 4)
    rt = make_compressor("powersgd", rank=2).round_trip([m, -m], ctx_at(), Communicator(2))
    assert np.max(np.abs(rt.aggregated)) == 0.0
    assert np.max(np.abs(rt.payload.p.T @ rt.payload.p - np.eye(2))) <= FP32
    ref = O.PowerSGD(2).round_trip([m, -m], O.CompressionContext(123), O.Communicator(2))
    assert np.max(np.abs(rt.payload.p - ref.payload.p)) <= 1e-6

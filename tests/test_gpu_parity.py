"""GPU parity: the sm_100a path against the CPU oracle (pinned to the reference)
and against the reference's own golden fixtures.

Tolerance (north_star, BASELINE.json): relative Frobenius error <= 1e-4 on
P-hat, Q-bar, M-hat and every error buffer e_w.  The oracle computes in float64
on the same fp32 inputs; the GPU computes in fp32 (FFMA, no TF32) with a float64
Gram-Schmidt.
"""

import os

import numpy as np
import pytest
import torch

from oracle import powersgd as O
from paper_1905_13727_b200 import ParamSpec, PowerSGDEngine, catalogs

pytestmark = pytest.mark.gpu

TOL = 1e-4


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def rel_e(e, e_ref, delta, full_rank):
    """Relative error of an error buffer.  When r_eff == min(n, m) the low-rank
    step is exact and e_ref is rounding noise (~1e-16 in float64), so the
    denominator is ||delta|| instead (the scale e is computed at)."""
    e_ref = np.asarray(e_ref, dtype=np.float64)
    den = np.linalg.norm(np.asarray(delta, dtype=np.float64)) if full_rank else np.linalg.norm(e_ref)
    return float(np.linalg.norm(np.asarray(e, dtype=np.float64) - e_ref) / (den if den > 0 else 1.0))


def np32(x):
    return np.asarray(x, dtype=np.float32)


def run_synced_step(specs, rank, world, seed=0, e_scale=0.5, step_idx=3, q_warm=True):
    """One engine step and one oracle step from the SAME state (g, e, Q), then
    the per-quantity relative errors."""
    ospecs = [O.ParamSpec(s.name, s.shape) for s in specs]
    eng = PowerSGDEngine(specs, rank, workers=world, seed=seed)
    comp = O.PowerSGD(rank)
    workers = [O.WorkerState(w) for w in range(world)]
    grads = [[None] * len(specs) for _ in range(world)]
    for i, s in enumerate(specs):
        for w in range(world):
            g = np32(O.derive_rng(seed, "grad", step_idx, w, i).standard_normal(s.shape))
            grads[w][i] = g
            eng.grad_view(i, w).copy_(torch.from_numpy(g))
        if s.is_bias:
            continue
        n, m = s.matrix_shape
        r = min(n, m, rank)
        if q_warm:
            q = np32(O.derive_rng(seed, "qwarm", i).standard_normal((m, r)))
            eng.q_view(i).copy_(torch.from_numpy(q))
            comp.q_memory[i] = q.astype(np.float64)
        for w in range(world):
            e = np32(e_scale * O.derive_rng(seed, "e", w, i).standard_normal((n, m)))
            eng.error_view(i, w).copy_(torch.from_numpy(e))
            workers[w].error[i] = e.astype(np.float64)
    deltas = {(w, i): grads[w][i].reshape(workers[w].error[i].shape).astype(np.float64) + workers[w].error[i]
              for w in range(world) for i in range(len(specs)) if not specs[i].is_bias}
    eng.step()
    torch.cuda.synchronize()
    updates, payloads = O.ef_step(workers, grads, ospecs, comp, O.Communicator(world), seed, step_idx)
    errs = {"p": 0.0, "q": 0.0, "mhat": 0.0, "e": 0.0, "bias": 0.0}
    for i, s in enumerate(specs):
        if s.is_bias:
            errs["bias"] = max(errs["bias"], rel(eng.update_view(i).cpu().numpy(), updates[i]))
            continue
        errs["p"] = max(errs["p"], rel(eng.p_view(i).cpu().numpy(), payloads[i].p))
        errs["q"] = max(errs["q"], rel(eng.q_view(i).cpu().numpy(), payloads[i].q))
        errs["mhat"] = max(errs["mhat"], rel(eng.update_view(i).cpu().numpy(), updates[i]))
        n, m = s.matrix_shape
        for w in range(world):
            errs["e"] = max(errs["e"], rel_e(eng.error_view(i, w).cpu().numpy(), workers[w].error[i],
                                             deltas[(w, i)], min(n, m, rank) == min(n, m)))
    return errs, eng


@pytest.mark.parametrize("rank", [1, 2, 4])
def test_resnet18_single_gpu_matches_oracle(rank):
    errs, _ = run_synced_step(list(catalogs.RESNET18.params), rank, 1)
    assert max(errs.values()) <= TOL, errs


def test_resnet18_two_simulated_workers_matches_oracle():
    # BASELINE.json configs[0]: the CPU reference's own workload
    errs, _ = run_synced_step(list(catalogs.RESNET18.params), 2, 2)
    assert max(errs.values()) <= TOL, errs


def test_resnet18_cold_start_seeded_q():
    errs, _ = run_synced_step(list(catalogs.RESNET18.params), 2, 1, e_scale=0.0, q_warm=False, step_idx=0)
    assert max(errs.values()) <= TOL, errs


def test_lstm_tall_path_matches_oracle():
    errs, eng = run_synced_step(list(catalogs.LSTM.params), 4, 1)
    assert eng.plan.info.n_tall == 7
    assert max(errs.values()) <= TOL, errs


def test_lstm_tall_path_three_workers():
    errs, _ = run_synced_step(list(catalogs.LSTM.params)[:3] + [catalogs.LSTM.params[-1]], 4, 3)
    assert max(errs.values()) <= TOL, errs


def test_stress_sampled_matrices_match_oracle():
    # configs[4] matrices are independent per step, so parity on a sample is exact parity
    specs = [ParamSpec(f"w{i}", (4096, 4096)) for i in range(3)]
    errs, _ = run_synced_step(specs, 8, 1)
    assert max(errs.values()) <= TOL, errs


def test_odd_shapes_and_rank_clamps():
    specs = [ParamSpec("a", (8, 6)), ParamSpec("b", (16, 3, 2, 2)), ParamSpec("bias", (10,)),
             ParamSpec("c", (3, 20)), ParamSpec("d", (513, 7)), ParamSpec("e", (5, 1)),
             ParamSpec("f", (700, 33)), ParamSpec("g", (1, 9)), ParamSpec("h", (1030, 1030)),
             ParamSpec("t", (900, 132)), ParamSpec("u", (96, 2056)), ParamSpec("v", (700, 130)),
             ParamSpec("bias2", (3,))]  # t: K4 column tiles (last tile 4 cols); u: K1 column tiles at r >= 8; v: K4 two-alignment tiles
    for rank, world in [(1, 1), (3, 1), (8, 2), (12, 1), (16, 3)]:
        errs, _ = run_synced_step(specs, rank, world)
        assert max(errs.values()) <= TOL, (rank, world, errs)


@pytest.mark.parametrize("case", ["r2_w1", "r4_w2", "r1_w3"])
def test_reference_golden_free_running(golden_dir, case):
    """Three free-running steps against the reference's own recorded outputs."""
    z = np.load(os.path.join(golden_dir, f"ef_steps_{case}.npz"))
    names = list(z["names"])
    specs = [ParamSpec(str(nm), tuple(int(x) for x in z[f"shape_{i}"])) for i, nm in enumerate(names)]
    world, rank, steps, seed = int(z["world"]), int(z["rank"]), int(z["steps"]), int(z["seed"])
    eng = PowerSGDEngine(specs, rank, workers=world, seed=seed)
    for t in range(steps):
        for w in range(world):
            for i in range(len(specs)):
                eng.grad_view(i, w).copy_(torch.from_numpy(z[f"s{t}_g_w{w}_p{i}"]))
        eng.step()
        for i, s in enumerate(specs):
            if s.is_bias:
                assert rel(eng.update_view(i).cpu(), z[f"s{t}_bias_p{i}"]) <= 1e-6
                continue
            assert rel(eng.p_view(i).cpu(), z[f"s{t}_phat_p{i}"]) <= TOL, (t, i)
            assert rel(eng.q_view(i).cpu(), z[f"s{t}_qbar_p{i}"]) <= TOL, (t, i)
            assert rel(eng.update_view(i).cpu().reshape(s.matrix_shape), z[f"s{t}_mhat_p{i}"]) <= TOL
            n, m = s.matrix_shape
            for w in range(world):
                delta = z[f"s{t}_g_w{w}_p{i}"].reshape(n, m).astype(np.float64) + z[f"s{t}_e_in_w{w}_p{i}"]
                assert rel_e(eng.error_view(i, w).cpu(), z[f"s{t}_e_w{w}_p{i}"], delta,
                             min(n, m, rank) == min(n, m)) <= TOL, (t, i, w)
        assert eng.stats.bits_allreduced == int(z[f"s{t}_bits"])
        assert eng.stats.decode_ops == int(z[f"s{t}_decode_ops"])
        assert eng.stats.compress_flops == int(z[f"s{t}_compress_flops"])


def test_bitwise_deterministic_and_graph_replay_identical():
    specs = list(catalogs.RESNET18.params)
    outs = []
    for use_graph in (False, False, True):
        eng = PowerSGDEngine(specs, 2, seed=1)
        for i in range(len(specs)):
            v = eng.grad_view(i)
            v.copy_(torch.randn(v.shape, generator=torch.Generator().manual_seed(i)))
        if use_graph:
            eng.capture()
        for _ in range(3):
            eng.step()
        outs.append((eng.work[0].clone(), eng.e[0].clone(), eng.Q.clone()))
    for a, b in zip(outs[0], outs[1]):
        assert torch.equal(a, b)
    for a, b in zip(outs[0], outs[2]):
        assert torch.equal(a, b)


def test_nonfinite_gradient_raises_and_leaves_state_untouched():
    from paper_1905_13727_b200 import NonFiniteGradient
    specs = list(catalogs.RESNET18.params)
    eng = PowerSGDEngine(specs, 2, workers=2)
    for w in range(2):
        for i in range(len(specs)):
            eng.grad_view(i, w).normal_()
    eng.step()
    e0, e1, q = eng.e[0].clone(), eng.e[1].clone(), eng.Q.clone()
    eng.grad_view(5, 1).view(-1)[17] = float("nan")
    with pytest.raises(NonFiniteGradient) as ei:
        eng.step()
    assert ei.value.param_name == specs[5].name and ei.value.worker == 1
    assert torch.equal(eng.e[0], e0) and torch.equal(eng.e[1], e1) and torch.equal(eng.Q, q)
    eng.grad_view(5, 1).view(-1)[17] = 0.0
    eng.grad_view(21, 0)[3] = float("inf")  # bias
    with pytest.raises(NonFiniteGradient) as ei:
        eng.step()
    assert ei.value.param_name == "bias_vectors" and ei.value.worker == 0


@pytest.mark.parametrize("rank,world", [(1, 1), (2, 2), (3, 1), (4, 1), (4, 3)])
def test_row_block_q_pass_shapes(rank, world):
    """k3_rq (the bulk-TMA row-block q pass of tall matrices with m = 2 mod 4,
    m <= 960, r <= 4): several row groups per column pair (m = 98, 130, 2, 6),
    Gram-space matrices whose P-hat k3_rq makes itself (n > 1024) and K2-MGS
    matrices whose P-hat it stages (n <= 1024), odd n, many matrices per CTA."""
    specs = [ParamSpec("g98", (1500, 98)), ParamSpec("b", (50,)), ParamSpec("o650", (3001, 650)),
             ParamSpec("v130", (700, 130)), ParamSpec("m2", (1030, 2)), ParamSpec("m6", (2000, 6)),
             ParamSpec("s18", (5000, 18)), ParamSpec("w", (64, 576))]
    errs, _ = run_synced_step(specs, rank, world)
    assert max(errs.values()) <= TOL, (rank, world, errs)


def test_row_block_q_pass_bitwise_deterministic():
    """Static row ranges per CTA and in-order slot sums: two runs from the same state agree bit for bit."""
    specs = [ParamSpec("o650", (3001, 650)), ParamSpec("g98", (1500, 98)), ParamSpec("b", (7,))]
    outs = []
    for _ in range(2):
        _, eng = run_synced_step(specs, 4, 1)
        outs.append([eng.update_view(i).cpu().numpy().copy() for i in range(len(specs))] +
                    [eng.q_view(i).cpu().numpy().copy() for i in (0, 1)] +
                    [eng.error_view(i, 0).cpu().numpy().copy() for i in (0, 1)])
    for a, b in zip(*outs):
        assert np.array_equal(a, b)

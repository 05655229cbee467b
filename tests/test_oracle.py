"""The CPU oracle (oracle/powersgd.py) is pinned to the reference itself:
golden fixtures written by tests/golden/make_golden.py from the reference's
own optimizer.step / PowerSGD / orthogonalize, plus the reference's own
known-answer tests."""

import os

import numpy as np
import pytest

from oracle import powersgd as O

GOLDEN_TRAIN = [  # pkg/tests/test_cli.py:10-17 (reference GOLDEN_TRAIN_CSV)
    (0, 39.31933055742294, 0, 0),
    (1, 38.53483587792976, 4352, 3072),
    (2, 37.10877043942111, 8704, 6144),
    (3, 35.33523873556888, 13056, 9216),
]


def load(golden_dir, name):
    return np.load(os.path.join(golden_dir, name), allow_pickle=False)


def specs_of(z):
    names = list(z["names"])
    return [O.ParamSpec(str(nm), tuple(int(x) for x in z[f"shape_{i}"])) for i, nm in enumerate(names)]


def test_golden_train_csv_exact():
    assert O.train_losses(3, 2, 1) == GOLDEN_TRAIN


@pytest.mark.parametrize("case", ["r2_w1", "r4_w2", "r1_w3"])
def test_oracle_matches_reference_ef_steps(golden_dir, case):
    z = load(golden_dir, f"ef_steps_{case}.npz")
    specs = specs_of(z)
    world, rank, steps, seed = int(z["world"]), int(z["rank"]), int(z["steps"]), int(z["seed"])
    comp = O.PowerSGD(rank)
    comm = O.Communicator(world)
    workers = [O.WorkerState(w) for w in range(world)]
    for t in range(steps):
        grads = [[z[f"s{t}_g_w{w}_p{i}"] for i in range(len(specs))] for w in range(world)]
        updates, payloads = O.ef_step(workers, grads, specs, comp, comm, seed, t)
        for i, s in enumerate(specs):
            if s.is_bias:
                np.testing.assert_allclose(updates[i], z[f"s{t}_bias_p{i}"], rtol=1e-14, atol=0)
                continue
            np.testing.assert_allclose(payloads[i].p, z[f"s{t}_phat_p{i}"], rtol=1e-12, atol=1e-13)
            np.testing.assert_allclose(payloads[i].q, z[f"s{t}_qbar_p{i}"], rtol=1e-12, atol=1e-12)
            np.testing.assert_allclose(updates[i].reshape(s.matrix_shape), z[f"s{t}_mhat_p{i}"],
                                       rtol=1e-12, atol=1e-12)
            for w in range(world):
                np.testing.assert_allclose(workers[w].error[i], z[f"s{t}_e_w{w}_p{i}"], rtol=1e-12,
                                           atol=1e-12)
        assert comm.stats.bits_allreduced == int(z[f"s{t}_bits"])
        assert comm.stats.decode_ops == int(z[f"s{t}_decode_ops"])
        assert comm.stats.compress_flops == int(z[f"s{t}_compress_flops"])


def test_oracle_orthogonalize_matches_reference(golden_dir):
    z = load(golden_dir, "orthogonalize.npz")
    keys = [k[3:] for k in z.files if k.startswith("in_")]
    assert len(keys) >= 8
    for k in keys:
        got = O.orthogonalize(z[f"in_{k}"])
        np.testing.assert_allclose(got, z[f"out_{k}"], rtol=1e-12, atol=1e-13, err_msg=k)


def test_oracle_tree_order_is_the_reference_tree():
    # pkg/tests/test_comm.py:25-37
    rng = np.random.default_rng(42)
    values = [rng.standard_normal(32) * (10.0 ** rng.integers(-8, 8)) for _ in range(8)]
    got = O.Communicator(8).all_reduce_mean([v.copy() for v in values])
    t01, t23, t45, t67 = values[0] + values[1], values[2] + values[3], values[4] + values[5], values[6] + values[7]
    assert np.array_equal(got, ((t01 + t23) + (t45 + t67)) / 8.0)
    assert O.tree_reduce([1, 2, 3, 4, 5], lambda a, b: (a, b)) == (((1, 2), (3, 4)), 5)


def test_oracle_degenerate_cases():
    # pkg/tests/test_linalg.py:72-97 and SPEC.md worked example M1 = -M2
    rng = O.derive_rng(505, "degenerate")
    base = rng.standard_normal(9)
    q = O.orthogonalize(np.column_stack([base, base.copy(), np.zeros(9)]))
    assert np.max(np.abs(q.T @ q - np.eye(3))) <= 1e-10
    mats = [np.arange(12.0).reshape(3, 4), -np.arange(12.0).reshape(3, 4)]
    trip = O.PowerSGD(2).round_trip(mats, O.CompressionContext(0), O.Communicator(2))
    assert np.max(np.abs(trip.aggregated)) == 0.0
    assert np.max(np.abs(trip.payload.p.T @ trip.payload.p - np.eye(2))) <= 1e-12


def test_catalog_sizes_match_survey():
    n_res = sum(np.prod(s.matrix_shape) for s in O.RESNET18 if not s.is_bias)
    n_lstm = sum(np.prod(s.matrix_shape) for s in O.LSTM if not s.is_bias)
    assert n_res == 11_164_352 and n_lstm == 28_904_850
    assert sum(s.shape[0] for s in O.RESNET18 if s.is_bias) == 9728

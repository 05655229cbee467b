"""GPU: the sibling low-rank compressors on the same kernels.

BestApproximation (compressors.py:400-438: four fresh power iterations, K1 /
K2+K3 / K5 per round) and UnbiasedRankK (:444-468: K1 sketch, K5 outer
products) through the drop-in API, against (a) the reference's own round trips
recorded in tests/golden/siblings.npz and (b) the reference's unit tests for
these classes (tests/test_compressors.py:185-225).  fp32 tolerance 1e-4
relative (north_star); accounting exact.
"""

import os

import numpy as np
import pytest

from oracle import powersgd as O
from paper_1905_13727_b200 import (BestApproximation, Communicator, CompressionContext, RandomProjection,
                                   UnbiasedRankK, decompress, make_compressor)

pytestmark = pytest.mark.gpu
TOL = 1e-4


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


@pytest.mark.parametrize("name", ["bestapprox", "unbiased"])
def test_siblings_match_reference_round_trips(golden_dir, name):
    z = np.load(os.path.join(golden_dir, "siblings.npz"))
    keys = sorted({k.rsplit("_", 1)[0] for k in z.files if k.startswith(name) and k.endswith("_agg")})
    for key in keys:
        world = int(key.split("_w")[1].split("_")[0])
        rank = int(key.split("_r")[1].split("_")[0])
        seed, pi, step = (int(x) for x in z[f"{key}_ctx"])
        mats = [z[f"{key}_in{w}"] for w in range(world)]
        comm = Communicator(world)
        trip = make_compressor(name, rank).round_trip(mats, CompressionContext(seed, pi, step), comm)
        assert rel(trip.aggregated, z[f"{key}_agg"]) <= TOL, key
        for w in range(world):
            assert rel(trip.locals[w], z[f"{key}_loc{w}"]) <= TOL, (key, w)
        p, q = (trip.payload.p, trip.payload.q) if name == "bestapprox" else (trip.payload.proj, trip.payload.u)
        assert rel(p, z[f"{key}_p"]) <= TOL and rel(q, z[f"{key}_q"]) <= TOL, key
        stats = [comm.stats.bits_allreduced, comm.stats.compress_flops, comm.stats.decode_ops]
        assert stats == list(z[f"{key}_stats"]), (key, stats)


def test_best_approximation_reaches_the_oracle_error():
    # reference tests/test_compressors.py:186-195
    rng = O.derive_rng(907, "bestapprox")
    u = rng.standard_normal((14, 3))
    v = rng.standard_normal((11, 3))
    mat = (u * np.array([8.0, 4.0, 0.5])) @ v.T
    payload = BestApproximation(2).compress(mat, CompressionContext(0))
    err = float(np.linalg.norm(mat - decompress(payload)))
    s = np.linalg.svd(mat, compute_uv=False)
    best = float(np.sqrt(np.sum(s[2:] ** 2)))
    assert err <= best * 1.001


def test_best_approximation_charges_four_rounds():
    # reference tests/test_compressors.py:198-202
    comm = Communicator(2)
    mats = [O.derive_rng(5, "w", w).standard_normal((8, 6)) for w in range(2)]
    BestApproximation(2).round_trip(mats, CompressionContext(0), comm)
    assert comm.stats.bits_allreduced == 4 * 32 * 2 * (8 + 6)


def test_unbiased_projection_uses_the_shared_stream():
    # reference tests/test_compressors.py:208-216 (proj within fp32 tolerance; u exact)
    mat = O.derive_rng(908, "unbiased").standard_normal((7, 5))
    ctx = CompressionContext(0, param_index=1, step=4)
    payload = UnbiasedRankK(2).compress(mat, ctx)
    u = ctx.rng("projection").standard_normal((5, 2)) / np.sqrt(2)
    assert isinstance(payload, RandomProjection)
    assert np.array_equal(payload.u, u)
    assert rel(payload.proj, mat @ u) <= TOL
    assert rel(decompress(payload), (mat @ u) @ u.T) <= TOL


def test_unbiased_projection_changes_with_step():
    comp = UnbiasedRankK(1)
    p0 = comp.compress(np.eye(4), CompressionContext(0, step=0))
    p1 = comp.compress(np.eye(4), CompressionContext(0, step=1))
    assert not np.array_equal(p0.u, p1.u)


def test_payload_bits_closed_forms():
    n, m, r = 6, 9, 2
    assert make_compressor("bestapprox", r).payload_bits(n, m) == 4 * 32 * r * (n + m)
    assert make_compressor("unbiased", r).payload_bits(n, m) == 32 * r * n
    assert make_compressor("powersgd", r).payload_bits(n, m) == 32 * r * (n + m)

"""Generate the golden fixtures that pin `oracle/powersgd.py` (and, through it,
the CUDA path) to the REFERENCE ITSELF.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It drives the reference's own `optimizer.step` (pkg/src/gradcomp/optimizer.py:98-135)
with its own `PowerSGD` (compressors.py:344-397) and `Communicator`
(comm.py:70-98), recording every round trip through spy subclasses, and writes
`tests/golden/ef_steps_*.npz` and `tests/golden/orthogonalize.npz`.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

from gradcomp.catalogs import ParamSpec  # noqa: E402
from gradcomp.comm import Communicator  # noqa: E402
from gradcomp.compressors import PowerSGD  # noqa: E402
from gradcomp.linalg import orthogonalize  # noqa: E402
from gradcomp.optimizer import OptimizerState, WorkerState, step  # noqa: E402
from gradcomp.seeding import derive_rng  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# shapes chosen to hit every kernel branch: m % 4 != 0, rank clamps (n < r,
# m < r), a bias between matrices (param_index counts it), tall and wide
SPECS = [
    ("a", (8, 6)),
    ("b", (16, 3, 2, 2)),
    ("bias0", (10,)),
    ("c", (3, 20)),
    ("d", (40, 32)),
    ("e", (5, 1)),
    ("bias1", (7,)),
    ("f", (70, 36)),
]


class SpyPowerSGD(PowerSGD):
    def __init__(self, rank):
        super().__init__(rank)
        self.trips = {}

    def round_trip(self, mats, ctx, comm):
        q_in = self._q_for(ctx, *mats[0].shape).copy()
        trip = super().round_trip(mats, ctx, comm)
        self.trips[ctx.param_index] = (q_in, trip)
        return trip


class SpyComm(Communicator):
    def __init__(self, w):
        super().__init__(w)
        self.means = []

    def all_reduce_mean(self, arrays, payload_bits=None):
        out = super().all_reduce_mean(arrays, payload_bits)
        self.means.append(out)
        return out


def grads_for(specs, step_idx, world, seed):
    return [[derive_rng(seed, "grad", step_idx, w, i).standard_normal(s.shape).astype(np.float32)
             for i, s in enumerate(specs)] for w in range(world)]


def ef_case(name, rank, world, steps, seed=0):
    specs = [ParamSpec(n, s) for n, s in SPECS]
    comp = SpyPowerSGD(rank)
    comm = SpyComm(world)
    params = [np.zeros(s.shape) for s in specs]
    opt = OptimizerState.init(params, 0.01, 0.9)
    workers = [WorkerState(w) for w in range(world)]
    out = {"rank": rank, "world": world, "steps": steps, "seed": seed,
           "names": np.array([n for n, _ in SPECS])}
    for i, s in enumerate(specs):
        out[f"shape_{i}"] = np.array(s.shape)
    for t in range(steps):
        grads = grads_for(specs, t, world, seed)
        comp.trips.clear()
        comm.means.clear()
        # EF state BEFORE this step, for single-step (re-synced) parity
        for w in range(world):
            for i, s in enumerate(specs):
                if not s.is_bias:
                    out[f"s{t}_e_in_w{w}_p{i}"] = workers[w].error_for(i, s.matrix_shape).copy()
        step(opt, workers, grads, specs, comp, comm, seed)
        for w in range(world):
            for i, s in enumerate(specs):
                out[f"s{t}_g_w{w}_p{i}"] = grads[w][i]
        for i, s in enumerate(specs):
            if s.is_bias:
                continue
            q_in, trip = comp.trips[i]
            out[f"s{t}_q_in_p{i}"] = q_in
            out[f"s{t}_phat_p{i}"] = trip.payload.p
            out[f"s{t}_qbar_p{i}"] = trip.payload.q
            out[f"s{t}_mhat_p{i}"] = trip.aggregated
            for w in range(world):
                out[f"s{t}_e_w{w}_p{i}"] = workers[w].error[i]
        # bias means in call order (world 1: copies; comm.py:92-93)
        bias_idx = [i for i, s in enumerate(specs) if s.is_bias]
        if world > 1:
            # the comm spy saw, per matrix, P then Q means, and one mean per bias
            k = 0
            for i, s in enumerate(specs):
                if s.is_bias:
                    out[f"s{t}_bias_p{i}"] = comm.means[k]
                    k += 1
                else:
                    k += 2
        else:
            for i in bias_idx:
                out[f"s{t}_bias_p{i}"] = grads[0][i].astype(np.float64)
        out[f"s{t}_bits"] = comm.stats.bits_allreduced
        out[f"s{t}_decode_ops"] = comm.stats.decode_ops
        out[f"s{t}_compress_flops"] = comm.stats.compress_flops
    np.savez_compressed(os.path.join(HERE, f"ef_steps_{name}.npz"), **out)


def orth_cases():
    out = {}
    rng = derive_rng(505, "golden_orth")
    cases = {
        "rand_12x1": rng.standard_normal((12, 1)),
        "rand_12x2": rng.standard_normal((12, 2)),
        "rand_64x5": rng.standard_normal((64, 5)),
        "rand_513x8": rng.standard_normal((513, 8)),
    }
    base = rng.standard_normal(9)
    cases["dup_zero_9x3"] = np.column_stack([base, base.copy(), np.zeros(9)])
    col = rng.standard_normal(7)
    cases["opposite_7x2"] = np.column_stack([col, -col])
    cases["ones_6x2"] = np.column_stack([np.ones(6), np.ones(6)])
    cases["zero_5x2"] = np.zeros((5, 2))
    cases["square_4x4"] = rng.standard_normal((4, 4))
    for k, p in cases.items():
        out[f"in_{k}"] = p
        out[f"out_{k}"] = orthogonalize(p.copy())
    np.savez_compressed(os.path.join(HERE, "orthogonalize.npz"), **out)


def sibling_cases():
    """The reference's own BestApproximation / UnbiasedRankK round trips
    (compressors.py:400-468 via make_compressor) on seeded worker matrices."""
    from gradcomp.compressors import CompressionContext, make_compressor
    out = {}
    shapes = [(8, 6), (3, 20), (40, 32), (65, 7)]
    for name in ("bestapprox", "unbiased"):
        for rank in (1, 2, 3):
            for world in (1, 2, 3):
                for si, (n, m) in enumerate(shapes):
                    key = f"{name}_r{rank}_w{world}_s{si}"
                    mats = [derive_rng(77, "sib", name, rank, world, si, w).standard_normal((n, m))
                            .astype(np.float32).astype(np.float64) for w in range(world)]
                    comp = make_compressor(name, rank=rank)
                    comm = Communicator(world)
                    ctx = CompressionContext(11, param_index=si, step=rank + world)
                    trip = comp.round_trip(mats, ctx, comm)
                    for w in range(world):
                        out[f"{key}_in{w}"] = mats[w]
                        out[f"{key}_loc{w}"] = trip.locals[w]
                    out[f"{key}_agg"] = trip.aggregated
                    if name == "bestapprox":
                        out[f"{key}_p"], out[f"{key}_q"] = trip.payload.p, trip.payload.q
                    else:
                        out[f"{key}_p"], out[f"{key}_q"] = trip.payload.proj, trip.payload.u
                    out[f"{key}_stats"] = np.array([comm.stats.bits_allreduced, comm.stats.compress_flops,
                                                    comm.stats.decode_ops])
                    out[f"{key}_ctx"] = np.array([11, si, rank + world])
    np.savez_compressed(os.path.join(HERE, "siblings.npz"), **out)


if __name__ == "__main__":
    ef_case("r2_w1", rank=2, world=1, steps=3)
    ef_case("r4_w2", rank=4, world=2, steps=3)
    ef_case("r1_w3", rank=1, world=3, steps=3)
    orth_cases()
    sibling_cases()
    print("wrote", sorted(f for f in os.listdir(HERE) if f.endswith(".npz")))

"""CPU ORACLE — test infrastructure only, never the product path.

A float64 numpy restatement of the reference's PowerSGD hot path
(`/root/reference/pkg/src/gradcomp`), used by `tests/`, `__graft_entry__.smoke()`
and the `cpu_baseline` / `--impl reference` legs of `bench.py` as the CHECKER
and the CPU baseline.  Nothing in `paper_1905_13727_b200/` imports this file.

Parity is PINNED: `tests/golden/make_golden.py` imports the reference itself (in
the build container) and writes `tests/golden/*.npz`; `tests/test_oracle.py`
checks this restatement against those fixtures and against the reference's own
known-answer tests (`pkg/tests/test_cli.py:10-17` GOLDEN_TRAIN_CSV,
`pkg/tests/test_comm.py:25-37` tree order, `pkg/tests/test_linalg.py:43-97`
degenerate Gram-Schmidt).

Every function cites the reference file:line it restates.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from math import prod

import numpy as np

FLOAT_BITS = 32                 # compressors.py:23
DEGENERATE_EPS = 1e-12          # linalg.py:15
GS_REPLACEMENT_TAG = 0x67736673  # linalg.py:17


class ContractViolation(ValueError):
    """linalg.py:20-21."""


class NonFiniteGradient(RuntimeError):
    """optimizer.py:31-38."""

    def __init__(self, param_name, worker):
        super().__init__(f"non-finite gradient for parameter {param_name!r} on worker {worker}")
        self.param_name = param_name
        self.worker = worker


# --------------------------------------------------------------------------- seeding

def derive_rng(seed, *labels):
    """seeding.py:11-24: SeedSequence([seed mod 2^64, *label entropies]) -> PCG64."""
    ent = [int(seed) & 0xFFFFFFFFFFFFFFFF]
    for lab in labels:
        if isinstance(lab, (int, np.integer)):
            if lab < 0:
                raise ValueError(f"labels must be non-negative, got {lab}")
            ent.append(int(lab))
        elif isinstance(lab, str):
            ent.append(int.from_bytes(lab.encode("utf-8"), "little"))
        else:
            raise TypeError(f"unsupported label type: {type(lab).__name__}")
    return np.random.default_rng(np.random.SeedSequence(ent))


# --------------------------------------------------------------------------- comm

@dataclass
class CommStats:
    """comm.py:23-48 (counters only)."""
    bits_allreduced: int = 0
    bits_gathered: int = 0
    decode_ops: int = 0
    compress_flops: int = 0


def tree_reduce(values, combine):
    """comm.py:51-67: pairwise fold level by level, odd element carried."""
    level = list(values)
    if not level:
        raise ValueError("tree_reduce needs at least one value")
    while len(level) > 1:
        paired = [combine(level[i], level[i + 1]) for i in range(0, len(level) - 1, 2)]
        if len(level) % 2:
            paired.append(level[-1])
        level = paired
    return level[0]


class Communicator:
    """comm.py:70-98: simulated W-worker all-reduce mean (tree sum, then / W)."""

    def __init__(self, world_size, stats=None):
        if world_size < 1:
            raise ValueError(f"world_size must be >= 1, got {world_size}")
        self.world_size = world_size
        self.stats = stats if stats is not None else CommStats()

    def all_reduce_mean(self, arrays, payload_bits=None):
        if len(arrays) != self.world_size:
            raise ValueError(f"expected {self.world_size} entries, got {len(arrays)}")
        if self.world_size == 1:          # comm.py:92-93, a free copy
            return arrays[0].copy()
        self.stats.bits_allreduced += 32 * arrays[0].size if payload_bits is None else payload_bits
        return tree_reduce(arrays, lambda a, b: a + b) / self.world_size


# --------------------------------------------------------------------------- linalg

def as_matrix(a, name="matrix"):
    """linalg.py:24-37."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise ContractViolation(f"{name} must be 2-d, got shape {a.shape}")
    if min(a.shape) < 1:
        raise ContractViolation(f"{name} has an empty dimension: {a.shape}")
    if not np.isfinite(a).all():
        raise ContractViolation(f"{name} contains non-finite entries")
    return a


def replacement_column(n, j, attempt):
    """linalg.py:54-58: seeded unit vector for a degenerate column."""
    v = np.random.default_rng(np.random.SeedSequence([GS_REPLACEMENT_TAG, j, attempt])).standard_normal(n)
    return v / np.sqrt(v @ v)


def orthogonalize(p):
    """linalg.py:61-90: in-order MODIFIED Gram-Schmidt (each projection uses the
    running column), degenerate columns replaced by `replacement_column`."""
    out = as_matrix(p, "orthogonalize input").copy()
    n, r = out.shape
    if r > n:
        raise ContractViolation(f"cannot orthonormalize {r} columns in R^{n}")
    for j in range(r):
        v = out[:, j]
        before = np.sqrt(v @ v)
        for i in range(j):
            v -= (out[:, i] @ v) * out[:, i]
        nrm = np.sqrt(v @ v)
        attempt = 0
        while nrm < DEGENERATE_EPS * (before + 1.0):
            v[:] = replacement_column(n, j, attempt)
            before = 1.0
            for i in range(j):
                v -= (out[:, i] @ v) * out[:, i]
            nrm = np.sqrt(v @ v)
            attempt += 1
        v /= nrm
    return out


def orthogonalize_flops(n, r):
    """linalg.py:93-99."""
    return 2 * n * r * r + 3 * n * r


# --------------------------------------------------------------------------- compressor

@dataclass
class CompressionContext:
    """compressors.py:27-45."""
    shared_seed: int
    param_index: int = 0
    step: int = 0

    def param_rng(self, label):
        return derive_rng(self.shared_seed, label, self.param_index)

    def rng(self, label):
        """compressors.py:38-40: stream tied to (seed, label, parameter, step)."""
        return derive_rng(self.shared_seed, label, self.param_index, self.step)


@dataclass
class LowRank:
    """compressors.py:59-67."""
    p: np.ndarray
    q: np.ndarray

    def bits(self):
        return FLOAT_BITS * (self.p.size + self.q.size)


@dataclass
class RoundTrip:
    """compressors.py:196-209."""
    aggregated: np.ndarray
    locals: list
    payload: object = None


def low_rank_iteration(mats, q, comm):
    """compressors.py:327-341."""
    n, r = mats[0].shape[0], q.shape[1]
    p = comm.all_reduce_mean([w @ q for w in mats], payload_bits=FLOAT_BITS * n * r)
    p_hat = orthogonalize(p)
    qs = [w.T @ p_hat for w in mats]
    q_bar = comm.all_reduce_mean(qs, payload_bits=FLOAT_BITS * q.shape[0] * r)
    return LowRank(p_hat, q_bar), qs


class PowerSGD:
    """compressors.py:344-397 (+ Compressor base :221-249)."""

    name = "powersgd"
    linear = True
    route = "allreduce"
    uses_error_feedback = True

    def __init__(self, rank=1):
        if rank < 1:
            raise ContractViolation(f"rank must be >= 1, got {rank}")
        self.rank = rank
        self.q_memory = {}

    def effective_rank(self, n, m):
        return min(n, m, self.rank)

    def initial_q(self, ctx, n, m):
        """compressors.py:362-367."""
        r = self.effective_rank(n, m)
        q = self.q_memory.get(ctx.param_index)
        if q is None or q.shape != (m, r):
            q = ctx.param_rng("warm_start_init").standard_normal((m, r))
        return q

    def round_trip(self, mats, ctx, comm):
        """compressors.py:369-379."""
        n, m = mats[0].shape
        comm.stats.compress_flops += len(mats) * self.compress_cost(n, m)
        payload, qs = low_rank_iteration(mats, self.initial_q(ctx, n, m), comm)
        self.q_memory[ctx.param_index] = payload.q
        comm.stats.decode_ops += 2 * n * m * payload.p.shape[1]   # decode_cost :176-182
        aggregated = payload.p @ payload.q.T                       # decompress :161
        return RoundTrip(aggregated, [payload.p @ qw.T for qw in qs], payload)

    def compress(self, m, ctx):
        return self.round_trip([m], ctx, Communicator(1)).payload

    def payload_bits(self, n, m):
        return FLOAT_BITS * self.effective_rank(n, m) * (n + m)

    def compress_cost(self, n, m):
        r = self.effective_rank(n, m)
        return 4 * n * m * r + orthogonalize_flops(n, r)


@dataclass
class RandomProjection:
    """compressors.py:70-78: proj = M u; u is seed-derived and costs no bits."""
    proj: np.ndarray
    u: np.ndarray

    def bits(self):
        return FLOAT_BITS * self.proj.size


class BestApproximation:
    """compressors.py:400-438: four fresh subspace iterations per call, no state."""

    name = "bestapprox"
    linear = True
    route = "allreduce"
    uses_error_feedback = True
    iterations = 4

    def __init__(self, rank=1):
        if rank < 1:
            raise ContractViolation(f"rank must be >= 1, got {rank}")
        self.rank = rank

    def round_trip(self, mats, ctx, comm):
        """compressors.py:407-420."""
        n, m = mats[0].shape
        comm.stats.compress_flops += len(mats) * self.compress_cost(n, m)
        rank = min(n, m, self.rank)
        q = ctx.rng("fresh_start").standard_normal((m, rank))
        payload, qs = None, None
        for _ in range(self.iterations):
            payload, qs = low_rank_iteration(mats, q, comm)
            q = payload.q
        comm.stats.decode_ops += 2 * n * m * payload.p.shape[1]
        return RoundTrip(payload.p @ payload.q.T, [payload.p @ qw.T for qw in qs], payload)

    def compress(self, m, ctx):
        return self.round_trip([m], ctx, Communicator(1)).payload

    def payload_bits(self, n, m):
        return self.iterations * FLOAT_BITS * min(n, m, self.rank) * (n + m)

    def compress_cost(self, n, m):
        r = min(n, m, self.rank)
        return self.iterations * (4 * n * m * r + orthogonalize_flops(n, r))


class UnbiasedRankK:
    """compressors.py:444-468 with the ReduceCompressor round trip (:255-269):
    proj_w = M_w u, u ~ N(0, 1/r) from the shared stream; aggregate mean(proj) u^T."""

    name = "unbiased"
    linear = True
    route = "allreduce"
    uses_error_feedback = True

    def __init__(self, rank=1):
        if rank < 1:
            raise ContractViolation(f"rank must be >= 1, got {rank}")
        self.rank = rank

    def compress(self, m, ctx):
        rows, cols = m.shape
        rank = min(rows, cols, self.rank)
        u = ctx.rng("projection").standard_normal((cols, rank)) / np.sqrt(rank)
        return RandomProjection(m @ u, u)

    def round_trip(self, mats, ctx, comm):
        n, m = mats[0].shape
        comm.stats.compress_flops += len(mats) * self.compress_cost(n, m)
        payloads = [self.compress(w, ctx) for w in mats]
        reduced = comm.all_reduce_mean([p.proj for p in payloads], payload_bits=self.payload_bits(n, m))
        combined = RandomProjection(reduced, payloads[0].u)
        comm.stats.decode_ops += 2 * n * m * combined.u.shape[1]   # decode_cost :183-185
        return RoundTrip(combined.proj @ combined.u.T, [p.proj @ p.u.T for p in payloads], combined)

    def payload_bits(self, n, m):
        return FLOAT_BITS * min(n, m, self.rank) * n

    def compress_cost(self, n, m):
        rank = min(n, m, self.rank)
        return 2 * n * m * rank + m * rank


# --------------------------------------------------------------------------- catalogs

@dataclass(frozen=True)
class ParamSpec:
    """catalogs.py:20-42: 1-d = bias; else (shape[0], prod(shape[1:]))."""
    name: str
    shape: tuple

    @property
    def is_bias(self):
        return len(self.shape) == 1

    @property
    def matrix_shape(self):
        return self.shape[0], prod(self.shape[1:])


def _specs(rows):
    return tuple(ParamSpec(n, s) for n, s in rows)


# catalogs.py:65-92 (order matters: param_index seeds Q)
RESNET18 = _specs([
    ("layer4.1.conv2", (512, 512, 3, 3)), ("layer4.0.conv2", (512, 512, 3, 3)),
    ("layer4.1.conv1", (512, 512, 3, 3)), ("layer4.0.conv1", (512, 256, 3, 3)),
    ("layer3.1.conv2", (256, 256, 3, 3)), ("layer3.1.conv1", (256, 256, 3, 3)),
    ("layer3.0.conv2", (256, 256, 3, 3)), ("layer3.0.conv1", (256, 128, 3, 3)),
    ("layer2.1.conv2", (128, 128, 3, 3)), ("layer2.1.conv1", (128, 128, 3, 3)),
    ("layer2.0.conv2", (128, 128, 3, 3)), ("layer4.0.shortcut.0", (512, 256, 1, 1)),
    ("layer2.0.conv1", (128, 64, 3, 3)), ("layer1.1.conv1", (64, 64, 3, 3)),
    ("layer1.1.conv2", (64, 64, 3, 3)), ("layer1.0.conv2", (64, 64, 3, 3)),
    ("layer1.0.conv1", (64, 64, 3, 3)), ("layer3.0.shortcut.0", (256, 128, 1, 1)),
    ("layer2.0.shortcut.0", (128, 64, 1, 1)), ("linear", (10, 512)),
    ("conv1", (64, 3, 3, 3)), ("bias_vectors", (9728,)),
])

# catalogs.py:96-109
LSTM = _specs([
    ("encoder", (28869, 650)),
    ("rnn.ih.l0", (2600, 650)), ("rnn.hh.l0", (2600, 650)),
    ("rnn.ih.l1", (2600, 650)), ("rnn.hh.l1", (2600, 650)),
    ("rnn.ih.l2", (2600, 650)), ("rnn.hh.l2", (2600, 650)),
    ("bias_vectors", (44469,)),
])


# --------------------------------------------------------------------------- EF step

@dataclass
class WorkerState:
    """optimizer.py:57-69 (EF memory only)."""
    index: int
    error: dict = field(default_factory=dict)

    def error_for(self, i, shape):
        if i not in self.error:
            self.error[i] = np.zeros(shape)
        return self.error[i]


def ef_step(workers, grads_per_worker, specs, compressor, comm, shared_seed, step_index,
            error_feedback=True):
    """optimizer.py:98-129 without the momentum/param update (:131-134), i.e.
    exactly the hot path: non-finite check, bias mean, then per matrix
    delta = g + e -> round_trip -> e = delta - local.  Returns the per-parameter
    aggregated updates (bias means and M-hat reshaped to the parameter shape)
    and the per-matrix RoundTrip payloads keyed by param_index."""
    for w, grads in enumerate(grads_per_worker):            # _check_finite :72-76
        for spec, g in zip(specs, grads):
            if not np.all(np.isfinite(g)):
                raise NonFiniteGradient(spec.name, w)
    world = len(workers)
    updates, payloads = [], {}
    for i, spec in enumerate(specs):
        if spec.is_bias:
            updates.append(comm.all_reduce_mean([grads_per_worker[w][i] for w in range(world)]))
            continue
        shape = spec.matrix_shape
        deltas = []
        for w in range(world):
            d = grads_per_worker[w][i].reshape(shape)
            if error_feedback:
                d = d + workers[w].error_for(i, shape)
            deltas.append(d)
        trip = compressor.round_trip(deltas, CompressionContext(shared_seed, i, step_index), comm)
        if error_feedback:
            for w in range(world):
                workers[w].error[i] = deltas[w] - trip.locals[w]
        payloads[i] = trip.payload
        updates.append(trip.aggregated.reshape(spec.shape))
    return updates, payloads


def momentum_update(params, buffers, updates, lr, momentum):
    """optimizer.py:131-134: m = momentum*m + u; x -= lr*(u + m)."""
    for x, buf, u in zip(params, buffers, updates):
        buf *= momentum
        buf += u
        x -= lr * (u + buf)


# --------------------------------------------------------------------------- desk problem (known-answer pin)

class LeastSquares:
    """problems.py:53-116 (noise 0) with the CLI defaults of problems.py:173-178
    (n=24, m=32, 256 samples).  `target_spectrum` is the conditioned instance of
    problems.py:78-86 (seeded orthonormal bases with exactly those singular
    values, mean-centred inputs, zero initial parameters) used by the reference's
    linearity check (verify.py:99-143).  Used to replay GOLDEN_TRAIN_CSV
    (pkg/tests/test_cli.py:10-17) and the linearity acceptance run."""

    def __init__(self, seed, n=24, m=32, n_samples=256, target_spectrum=None):
        rng = derive_rng(seed, "data")
        inputs = rng.standard_normal((n_samples, m))
        if target_spectrum is not None:                      # problems.py:78-86
            sig = tuple(float(x) for x in target_spectrum)
            inputs = inputs - inputs.mean(axis=0)
            u = np.linalg.qr(rng.standard_normal((n, n)))[0][:, :len(sig)]
            v = np.linalg.qr(rng.standard_normal((m, m)))[0][:, :len(sig)]
            w_true = (u * sig) @ v.T
        else:
            w_true = rng.standard_normal((n, m)) / np.sqrt(m)
        c_true = rng.standard_normal(n) * 0.5
        self.inputs = inputs
        self.targets = inputs @ w_true.T + c_true
        self.specs = [ParamSpec("weight", (n, m)), ParamSpec("bias", (n,))]
        self.seed = seed
        self.n_samples = n_samples
        self.target_spectrum = target_spectrum

    def init_params(self):                      # problems.py:28-34, :88-91
        if self.target_spectrum is not None:
            return [np.zeros(s.shape) for s in self.specs]
        rng = derive_rng(self.seed, "param_init")
        return [rng.standard_normal(s.shape) / np.sqrt(s.shape[-1] if not s.is_bias else 1)
                for s in self.specs]

    def loss(self, params, idx=slice(None)):    # problems.py:103-107
        w, c = params
        resid = self.inputs[idx] @ w.T + c - self.targets[idx]
        return float(np.sum(resid * resid) / (2 * resid.shape[0]))

    def gradients(self, params, idx=slice(None)):   # problems.py:109-115
        w, c = params
        a = self.inputs[idx]
        resid = a @ w.T + c - self.targets[idx]
        s = 1.0 / resid.shape[0]
        return [s * (resid.T @ a), s * np.sum(resid, axis=0)]

    def worker_gradients(self, params, w, world):   # problems.py:36-50
        per = self.n_samples // world
        return self.gradients(params, slice(w * per, (w + 1) * per))


def train_params(prob, steps, workers, seed, rank=2, lr=0.01, momentum=0.9):
    """train.py:78-139 for powersgd on `prob`: the final parameters."""
    comp = PowerSGD(rank)
    comm = Communicator(workers)
    params = prob.init_params()
    bufs = [np.zeros_like(p) for p in params]
    ws = [WorkerState(w) for w in range(workers)]
    for t in range(steps):
        grads = [prob.worker_gradients(params, w, workers) for w in range(workers)]
        updates, _ = ef_step(ws, grads, prob.specs, comp, comm, seed, t)
        momentum_update(params, bufs, updates, lr, momentum)
    return params


def train_losses(steps, workers, seed, rank=2, lr=0.01, momentum=0.9):
    """train.py:78-139 for powersgd: returns [(step, loss, bits, decode_ops)]."""
    prob = LeastSquares(seed)
    comp = PowerSGD(rank)
    comm = Communicator(workers)
    params = prob.init_params()
    bufs = [np.zeros_like(p) for p in params]
    ws = [WorkerState(w) for w in range(workers)]
    rows = [(0, prob.loss(params), 0, 0)]
    for t in range(steps):
        grads = [prob.worker_gradients(params, w, workers) for w in range(workers)]
        updates, _ = ef_step(ws, grads, prob.specs, comp, comm, seed, t)
        momentum_update(params, bufs, updates, lr, momentum)
        rows.append((t + 1, prob.loss(params),
                     comm.stats.bits_allreduced + comm.stats.bits_gathered, comm.stats.decode_ops))
    return rows

"""Drop-in for the reference's compressor plug-in API, backed by the B200 kernels.

Mirrors compressors.py:27-67 (CompressionContext, LowRank), :156-209
(decompress, decode_cost, RoundTrip), :221-249 (Compressor), :344-397
(PowerSGD) and :682-707 (registry / make_compressor) — same names, argument
meaning, accounting and errors.  Inputs may be numpy arrays (returned as
float64 numpy, like the reference) or CUDA tensors (returned as fp32 CUDA
tensors).  All arithmetic runs in the sm_100a kernels of libpsgd_b200.so.

`PowerSGD.round_trip(mats, ctx, comm)` with a `Communicator(W)` runs the
reference's simulated W-worker model on one GPU; with a
`DistributedCommunicator`, `mats` is this rank's single matrix and the two
all-reduces go over NCCL.  For whole models use `engine.PowerSGDEngine`, which
runs every parameter in one grouped kernel sequence.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .comm import Communicator, tree_mean_
from .linalg import ContractViolation
from .plan import Plan, ptr, stream_ptr
from .seeding import derive_rng

FLOAT_BITS = 32


@dataclass
class CompressionContext:
    """compressors.py:27-45."""

    shared_seed: int
    param_index: int = 0
    step: int = 0

    def rng(self, label):
        return derive_rng(self.shared_seed, label, self.param_index, self.step)

    def param_rng(self, label):
        return derive_rng(self.shared_seed, label, self.param_index)


@dataclass
class LowRank:
    """p @ q.T with orthonormal p columns (compressors.py:59-67)."""

    p: object  # n x r
    q: object  # m x r

    def bits(self):
        return FLOAT_BITS * (_numel(self.p) + _numel(self.q))


@dataclass
class RoundTrip:
    """compressors.py:196-209."""

    aggregated: object
    locals: list
    payload: object = None


def _numel(x):
    return x.numel() if isinstance(x, torch.Tensor) else int(np.asarray(x).size)


def _to_dev(x, device):
    if isinstance(x, torch.Tensor):
        return x.detach().to(device=device, dtype=torch.float32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64), dtype=np.float32)).to(device)


def _out(t, as_numpy):
    return t.double().cpu().numpy() if as_numpy else t


_PLANS = {}


def _plan(n, m, rank, world, device):
    key = (n, m, rank, world, str(device))
    pl = _PLANS.get(key)
    if pl is None:
        pl = _PLANS[key] = Plan([(n, m)], rank, world, 0, device)
    return pl


def decompress(payload, device=None):
    """compressors.py:156-173 for the low-rank payload: p @ q.T in the K5 kernel."""
    if not isinstance(payload, LowRank):
        raise TypeError(f"unknown payload type: {type(payload).__name__}")
    as_np = not isinstance(payload.p, torch.Tensor)
    dev = torch.device(device) if device is not None else (
        payload.p.device if not as_np else torch.device("cuda", torch.cuda.current_device()))
    p = _to_dev(payload.p, dev)
    q = _to_dev(payload.q, dev)
    n, r = p.shape
    m = q.shape[0]
    pl = _plan(n, m, r, 1, dev)
    pb = torch.zeros(pl.p_elems, dtype=torch.float32, device=dev)
    qb = torch.zeros(pl.q_elems, dtype=torch.float32, device=dev)
    pl.p_view(pb, 0).copy_(p)
    pl.q_view(qb, 0).copy_(q)
    out = torch.empty(pl.flat_elems, dtype=torch.float32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().psgd_decompress(pl.handle, ptr(pb), ptr(qb), 1, None, ptr(out), ptr(status),
                                              stream_ptr()), "psgd_decompress")
    return _out(pl.matrix_view(out, 0).clone(), as_np)


def decode_cost(payload):
    """compressors.py:176-182 (low-rank payload)."""
    if not isinstance(payload, LowRank):
        raise TypeError(f"unknown payload type: {type(payload).__name__}")
    n, r = tuple(payload.p.shape)
    return 2 * n * int(payload.q.shape[0]) * r


class Compressor:
    """compressors.py:221-249."""

    name = None
    linear = None
    route = None
    uses_error_feedback = True

    def __init__(self, rank=1):
        if rank < 1:
            raise ContractViolation(f"rank must be >= 1, got {rank}")
        self.rank = rank

    def compress(self, m, ctx):
        raise NotImplementedError

    def payload_bits(self, n, m):
        raise NotImplementedError

    def compress_cost(self, n, m):
        raise NotImplementedError

    def round_trip(self, mats, ctx, comm):
        raise NotImplementedError

    def _charge_compress(self, comm, n, m, workers):
        comm.stats.compress_flops += workers * self.compress_cost(n, m)


class PowerSGD(Compressor):
    """Rank-r compression by one warm-started power-iteration step
    (compressors.py:344-397).  `q_memory[param_index]` holds the fp32 Q-bar of
    the last step on the device (the reference stores it unnormalised, :373)."""

    name = "powersgd"
    linear = True
    route = "allreduce"
    uses_error_feedback = True

    def __init__(self, rank=1, device=None):
        super().__init__(rank)
        self.q_memory = {}
        self.device = device

    def effective_rank(self, n, m):
        return min(n, m, self.rank)

    def _q_for(self, ctx, n, m, device):
        r = self.effective_rank(n, m)
        q = self.q_memory.get(ctx.param_index)
        if q is None or tuple(q.shape) != (m, r):
            q = ctx.param_rng("warm_start_init").standard_normal((m, r))
        return _to_dev(q, device)

    def round_trip(self, mats, ctx, comm):
        """compressors.py:369-379 on the GPU."""
        as_np = not isinstance(mats[0], torch.Tensor)
        if len(mats) == 0:
            raise ValueError("round_trip needs at least one worker matrix")
        dist = bool(getattr(comm, "distributed", False))
        if not dist and len(mats) != comm.world_size:
            raise ValueError(f"expected {comm.world_size} entries, got {len(mats)}")
        if dist and len(mats) != 1:
            raise ValueError("a distributed worker passes its own matrix only")
        dev = (torch.device(self.device) if self.device is not None else
               (mats[0].device if not as_np else torch.device("cuda", torch.cuda.current_device())))
        ds = [_to_dev(x, dev) for x in mats]
        if ds[0].dim() != 2 or min(ds[0].shape) < 1:
            raise ContractViolation(f"matrix must be 2-d and non-empty, got {tuple(ds[0].shape)}")
        n, m = ds[0].shape
        W = len(ds)
        world = comm.world_size
        self._charge_compress(comm, n, m, W)
        r = self.effective_rank(n, m)
        pl = _plan(n, m, self.rank, world, dev)
        lib = _lib.lib()
        sp = stream_ptr()
        h = pl.handle
        f32 = dict(dtype=torch.float32, device=dev)
        q_in = torch.zeros(pl.q_elems, **f32)
        pl.q_view(q_in, 0).copy_(self._q_for(ctx, n, m, dev))
        status = torch.zeros(1, dtype=torch.int32, device=dev)
        repl = pl.repl_table()
        phat = torch.zeros(pl.p_elems, **f32)
        works, ps = [], []
        with torch.cuda.device(dev):
            for d in ds:       # low_rank_iteration :336 (delta comes in already EF-added)
                g = torch.zeros(pl.flat_elems, **f32)
                pl.matrix_view(g, 0).copy_(d)
                w = torch.empty(pl.flat_elems, **f32)
                p = torch.zeros(pl.p_elems, **f32)
                _lib.check(lib.psgd_ef_p(h, ptr(g), None, ptr(w), ptr(q_in), ptr(p), ptr(phat), ptr(repl), None,
                                         ptr(status), sp), "psgd_ef_p")
                works.append(w)
                ps.append(p)
            if dist:                      # :337
                comm.charge_allreduce(FLOAT_BITS * n * r)
                comm.all_reduce_sum_(ps[0])
                pm, div = ps[0], world
            elif W > 1:
                comm.charge_allreduce(FLOAT_BITS * n * r)
                pm, div = torch.empty_like(ps[0]), 1
                tree_mean_(ps, pm)
            else:
                pm, div = ps[0], 1
            qws, escratch = [], torch.empty(pl.flat_elems, **f32)
            for w in works:               # :338-339 (GS, q_w) and the EF locals (:376-378)
                qw = torch.zeros(pl.q_elems, **f32)
                _lib.check(lib.psgd_q_ef(h, ptr(w), ptr(pm), div, ptr(repl), ptr(phat), ptr(qw),
                                         ptr(escratch), None, ptr(status), sp), "psgd_q_ef")
                qws.append(qw)
            if world == 1:
                qbar = qws[0]
                agg = works[0]            # K3 wrote M-hat == local (W=1)
                locs = [agg.clone()]
            else:                         # :340, :375
                comm.charge_allreduce(FLOAT_BITS * m * r)
                if dist:
                    qbar = qws[0].clone()
                    comm.all_reduce_sum_(qbar)
                    qdiv = world
                else:
                    qbar = torch.empty_like(qws[0])
                    tree_mean_(qws, qbar)
                    qdiv = 1
                agg = torch.empty(pl.flat_elems, **f32)
                qstore = torch.zeros(pl.q_elems, **f32)
                _lib.check(lib.psgd_decompress(h, ptr(phat), ptr(qbar), qdiv, ptr(qstore), ptr(agg),
                                               ptr(status), sp), "psgd_decompress")
                if qdiv != 1:
                    qbar = qstore
                locs = []
                for qw in qws:
                    loc = torch.empty(pl.flat_elems, **f32)
                    _lib.check(lib.psgd_decompress(h, ptr(phat), ptr(qw), 1, None, ptr(loc), ptr(status), sp),
                               "psgd_decompress")
                    locs.append(loc)
        st = int(status.item())
        if st & (_lib.STATUS_NONFINITE_GRAD | _lib.STATUS_NONFINITE_P):
            raise ContractViolation("orthogonalize input contains non-finite entries")
        if st & _lib.STATUS_REPLACEMENT:
            raise RuntimeError("Gram-Schmidt needed more than one replacement draw")
        q_new = pl.q_view(qbar, 0).contiguous()
        self.q_memory[ctx.param_index] = q_new           # :373
        comm.stats.decode_ops += 2 * n * m * r           # :374
        payload = LowRank(_out(pl.p_view(phat, 0).clone(), as_np), _out(q_new, as_np))
        return RoundTrip(_out(pl.matrix_view(agg, 0).clone(), as_np),
                         [_out(pl.matrix_view(x, 0).clone(), as_np) for x in locs], payload)

    def compress(self, m, ctx):
        """Single-worker fused round; updates the warm-start memory (:381-384)."""
        return self.round_trip([m], ctx, Communicator(1)).payload

    def payload_bits(self, n, m):
        return FLOAT_BITS * self.effective_rank(n, m) * (n + m)

    def compress_cost(self, n, m):
        r = self.effective_rank(n, m)
        return 4 * n * m * r + 2 * n * r * r + 3 * n * r


COMPRESSORS = {PowerSGD.name: PowerSGD}


def make_compressor(name, rank=1):
    """compressors.py:703-707 (only the PowerSGD hot path is B200-native here)."""
    if name not in COMPRESSORS:
        raise ContractViolation(f"unknown compressor {name!r}; choose from {sorted(COMPRESSORS)}")
    return COMPRESSORS[name](rank=rank)

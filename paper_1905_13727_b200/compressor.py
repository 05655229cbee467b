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


def _raise_status(st):
    """The reference's errors for a device status word (linalg.py:35-36, :82-88)."""
    if st & (_lib.STATUS_NONFINITE_GRAD | _lib.STATUS_NONFINITE_P):
        raise ContractViolation("orthogonalize input contains non-finite entries")
    if st & _lib.STATUS_REPLACEMENT:
        raise RuntimeError(f"Gram-Schmidt needed more than {_lib.REPL_ATTEMPTS} replacement draws for a column")


def _plan(n, m, rank, world, device):
    key = (n, m, rank, world, str(device))
    pl = _PLANS.get(key)
    if pl is None:
        pl = _PLANS[key] = Plan([(n, m)], rank, world, 0, device)
    return pl


@dataclass
class RandomProjection:
    """proj = M @ u for a seed-derived u; u costs no bits (compressors.py:70-78)."""

    proj: object  # n x r
    u: object     # m x r

    def bits(self):
        return FLOAT_BITS * _numel(self.proj)


def decompress(payload, device=None):
    """compressors.py:156-173 for the low-rank payloads: p @ q.T (LowRank) or
    proj @ u.T (RandomProjection), in the K5 kernel."""
    if isinstance(payload, LowRank):
        pp, qq = payload.p, payload.q
    elif isinstance(payload, RandomProjection):
        pp, qq = payload.proj, payload.u
    else:
        raise TypeError(f"unknown payload type: {type(payload).__name__}")
    as_np = not isinstance(pp, torch.Tensor)
    dev = torch.device(device) if device is not None else (
        pp.device if not as_np else torch.device("cuda", torch.cuda.current_device()))
    p = _to_dev(pp, dev)
    q = _to_dev(qq, dev)
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
    """compressors.py:176-185 (low-rank payloads)."""
    if isinstance(payload, LowRank):
        n, r = tuple(payload.p.shape)
        return 2 * n * int(payload.q.shape[0]) * r
    if isinstance(payload, RandomProjection):
        n, r = tuple(payload.proj.shape)
        return 2 * n * int(payload.u.shape[0]) * r
    raise TypeError(f"unknown payload type: {type(payload).__name__}")


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


class _RoundTripWork:
    """Device and pinned-host buffers of one round-trip shape (n, m, W, world,
    device), allocated once and reused by every later call with that shape: a
    per-parameter drop-in call makes no allocations, one H2D copy per worker
    matrix, one D2H copy per output and (numpy mode) one stream synchronisation."""

    def __init__(self, n, m, rank, W, world, dev, host):
        self.pl = pl = _plan(n, m, rank, world, dev)
        f32 = dict(dtype=torch.float32, device=dev)
        self.r = min(n, m, rank)
        self.g = [torch.zeros(pl.flat_elems, **f32) for _ in range(W)]
        self.works = [torch.zeros(pl.flat_elems, **f32) for _ in range(W)]
        self.ps = [torch.zeros(pl.p_elems, **f32) for _ in range(W)]
        self.pm = torch.zeros(pl.p_elems, **f32)
        self.phat = torch.zeros(pl.p_elems, **f32)
        self.q_in = torch.zeros(pl.q_elems, **f32)
        self.qws = [torch.zeros(pl.q_elems, **f32) for _ in range(W)]
        self.qbar = torch.zeros(pl.q_elems, **f32)
        self.qstore = torch.zeros(pl.q_elems, **f32)
        self.escratch = torch.empty(pl.flat_elems, **f32)
        self.agg = torch.zeros(pl.flat_elems, **f32)
        self.locs = [torch.zeros(pl.flat_elems, **f32) for _ in range(W)] if world > 1 else []
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.repl = pl.repl_table()
        if host:  # pinned staging for numpy inputs / outputs
            pin = dict(dtype=torch.float32, pin_memory=True)
            self.h_in = [torch.empty((n, m), **pin) for _ in range(W)]
            self.h_agg = torch.empty((n, m), **pin)
            self.h_locs = [torch.empty((n, m), **pin) for _ in range(W)] if world > 1 else []
            self.h_p = torch.empty((n, self.r), **pin)
            self.h_q = torch.empty((m, self.r), **pin)
            self.h_st = torch.zeros(1, dtype=torch.int32, pin_memory=True)


class PowerSGD(Compressor):
    """Rank-r compression by one warm-started power-iteration step
    (compressors.py:344-397).  `q_memory[param_index]` holds Q-bar of the last
    step, unnormalised (:373): a float64 numpy array when the round trip was
    called with numpy matrices (as the reference), an fp32 CUDA tensor when it
    was called with CUDA tensors.  A device mirror of each stored Q-bar avoids
    re-uploading it on the next step.

    CUDA-tensor calls never synchronise: a non-finite input or an exhausted
    replacement table is recorded on the device and raised by `check()` (the
    grouped optimizer loop calls it once per step); numpy calls raise
    immediately, like the reference."""

    name = "powersgd"
    linear = True
    route = "allreduce"
    uses_error_feedback = True

    def __init__(self, rank=1, device=None):
        super().__init__(rank)
        self.q_memory = {}
        self.device = device
        self._work = {}
        self._q_dev = {}     # param_index -> (the q_memory object it mirrors, device fp32 m x r)
        self._sticky = {}    # device -> int32 status accumulated by tensor-mode calls

    def effective_rank(self, n, m):
        return min(n, m, self.rank)

    def _q_for(self, ctx, n, m, device):
        r = self.effective_rank(n, m)
        q = self.q_memory.get(ctx.param_index)
        if q is None or tuple(q.shape) != (m, r):
            q = ctx.param_rng("warm_start_init").standard_normal((m, r))
        mirror = self._q_dev.get(ctx.param_index)
        if mirror is not None and mirror[0] is q and mirror[1].device == device:
            return mirror[1]
        return _to_dev(q, device)

    def _ws(self, n, m, W, world, dev, host):
        key = (n, m, W, world, str(dev), host)
        w = self._work.get(key)
        if w is None:
            w = self._work[key] = _RoundTripWork(n, m, self.rank, W, world, dev, host)
        return w

    def check(self):
        """Raise what the reference would for the tensor-mode calls since the last check."""
        for dev, st in list(self._sticky.items()):
            v = int(st.item())
            st.zero_()
            _raise_status(v)

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
        shp = tuple(np.shape(mats[0]) if as_np else mats[0].shape)
        if len(shp) != 2 or min(shp) < 1:
            raise ContractViolation(f"matrix must be 2-d and non-empty, got {shp}")
        n, m = shp
        W = len(mats)
        world = comm.world_size
        self._charge_compress(comm, n, m, W)
        r = self.effective_rank(n, m)
        ws = self._ws(n, m, W, world, dev, as_np)
        pl = ws.pl
        lib = _lib.lib()
        h = pl.handle
        with torch.cuda.device(dev):
            sp = stream_ptr()
            for w, x in enumerate(mats):  # the worker matrices (delta: EF already added by the caller)
                if as_np:
                    np.copyto(ws.h_in[w].numpy(), np.asarray(x), casting="unsafe")
                    pl.matrix_view(ws.g[w], 0).view(n, m).copy_(ws.h_in[w], non_blocking=True)
                else:
                    pl.matrix_view(ws.g[w], 0).view(n, m).copy_(x.detach())
            pl.q_view(ws.q_in, 0).copy_(self._q_for(ctx, n, m, dev))
            for w in range(W):           # low_rank_iteration :336
                _lib.check(lib.psgd_ef_p(h, ptr(ws.g[w]), None, ptr(ws.works[w]), ptr(ws.q_in), ptr(ws.ps[w]),
                                         None, ptr(ws.status), sp), "psgd_ef_p")
            if dist:                      # :337
                comm.charge_allreduce(FLOAT_BITS * n * r)
                comm.all_reduce_sum_(ws.ps[0])
                pm, div = ws.ps[0], world
            elif W > 1:
                comm.charge_allreduce(FLOAT_BITS * n * r)
                tree_mean_(ws.ps, ws.pm)
                pm, div = ws.pm, 1
            else:
                pm, div = ws.ps[0], 1
            for w in range(W):            # :338-339 (GS, q_w) and the EF locals (:376-378)
                _lib.check(lib.psgd_q_ef(h, ptr(ws.works[w]), ptr(pm), div, ptr(ws.repl), ptr(ws.phat),
                                         ptr(ws.qws[w]), ptr(ws.escratch), None, ptr(ws.status), sp), "psgd_q_ef")
            if world == 1:
                qbar, agg, locs = ws.qws[0], ws.works[0], [ws.works[0]]  # K3 wrote M-hat == local (W=1)
            else:                         # :340, :375
                comm.charge_allreduce(FLOAT_BITS * m * r)
                if dist:
                    ws.qbar.copy_(ws.qws[0])
                    comm.all_reduce_sum_(ws.qbar)
                    qsum, qdiv = ws.qbar, world
                else:
                    tree_mean_(ws.qws, ws.qbar)
                    qsum, qdiv = ws.qbar, 1
                _lib.check(lib.psgd_decompress(h, ptr(ws.phat), ptr(qsum), qdiv, ptr(ws.qstore), ptr(ws.agg),
                                               ptr(ws.status), sp), "psgd_decompress")
                qbar = ws.qstore if qdiv != 1 else ws.qbar
                agg = ws.agg
                for w in range(W):
                    _lib.check(lib.psgd_decompress(h, ptr(ws.phat), ptr(ws.qws[w]), 1, None, ptr(ws.locs[w]),
                                                   ptr(ws.status), sp), "psgd_decompress")
                locs = ws.locs
            comm.stats.decode_ops += 2 * n * m * r           # :374
            if not as_np:  # device results; errors surface at check()
                st = self._sticky.get(dev)
                if st is None:
                    st = self._sticky[dev] = torch.zeros(1, dtype=torch.int32, device=dev)
                st.bitwise_or_(ws.status)
                q_new = pl.q_view(qbar, 0).clone()
                self.q_memory[ctx.param_index] = q_new       # :373
                self._q_dev[ctx.param_index] = (q_new, q_new)
                payload = LowRank(pl.p_view(ws.phat, 0).clone(), q_new)
                return RoundTrip(pl.matrix_view(agg, 0).view(n, m).clone(),
                                 [pl.matrix_view(x, 0).view(n, m).clone() for x in locs], payload)
            # numpy: every output copied out, one synchronisation, the status checked before anything is stored
            ws.h_agg.copy_(pl.matrix_view(agg, 0).view(n, m), non_blocking=True)
            if world > 1:
                for w in range(W):
                    ws.h_locs[w].copy_(pl.matrix_view(locs[w], 0).view(n, m), non_blocking=True)
            ws.h_p.copy_(pl.p_view(ws.phat, 0), non_blocking=True)
            ws.h_q.copy_(pl.q_view(qbar, 0), non_blocking=True)
            ws.h_st.copy_(ws.status, non_blocking=True)
            q_keep = pl.q_view(qbar, 0).clone()
            torch.cuda.current_stream().synchronize()
        _raise_status(int(ws.h_st[0]))
        q_new = ws.h_q.numpy().astype(np.float64)
        self.q_memory[ctx.param_index] = q_new               # :373
        self._q_dev[ctx.param_index] = (q_new, q_keep)
        agg_np = ws.h_agg.numpy().astype(np.float64)
        if world == 1:  # the local IS the aggregate at W = 1: a read-only view instead of an 11M-element copy
            loc = agg_np.view()
            loc.flags.writeable = False
            locs_np = [loc]
        else:
            locs_np = [x.numpy().astype(np.float64) for x in ws.h_locs]
        return RoundTrip(agg_np, locs_np, LowRank(ws.h_p.numpy().astype(np.float64), q_new))

    def compress(self, m, ctx):
        """Single-worker fused round; updates the warm-start memory (:381-384)."""
        return self.round_trip([m], ctx, Communicator(1)).payload

    def payload_bits(self, n, m):
        return FLOAT_BITS * self.effective_rank(n, m) * (n + m)

    def compress_cost(self, n, m):
        r = self.effective_rank(n, m)
        return 4 * n * m * r + 2 * n * r * r + 3 * n * r


# --------------------------------------------------------------------------- siblings on the same kernels

def _device_of(mats, device):
    if device is not None:
        return torch.device(device)
    if isinstance(mats[0], torch.Tensor):
        return mats[0].device
    return torch.device("cuda", torch.cuda.current_device())


def _check_mats(mats, comm):
    if len(mats) == 0:
        raise ValueError("round_trip needs at least one worker matrix")
    dist = bool(getattr(comm, "distributed", False))
    if not dist and len(mats) != comm.world_size:
        raise ValueError(f"expected {comm.world_size} entries, got {len(mats)}")
    if dist and len(mats) != 1:
        raise ValueError("a distributed worker passes its own matrix only")
    return dist


class _Rounds:
    """low_rank_iteration (compressors.py:327-341) on the device for W worker
    matrices, as many rounds as asked.  The plan has exchange semantics (K3 writes
    q_w and e, never M-hat), so delta survives every round."""

    def __init__(self, ds, comm, rank, dev):
        n, m = ds[0].shape
        self.n, self.m, self.dev, self.comm = n, m, dev, comm
        self.dist = bool(getattr(comm, "distributed", False))
        self.world = comm.world_size
        self.pl = pl = _plan(n, m, rank, max(2, self.world), dev)
        f32 = dict(dtype=torch.float32, device=dev)
        self.f32 = f32
        self.works = []
        for d in ds:
            w = torch.zeros(pl.flat_elems, **f32)
            pl.matrix_view(w, 0).copy_(d)
            self.works.append(w)
        self.scratch = torch.empty(pl.flat_elems, **f32)
        self.escratch = torch.empty(pl.flat_elems, **f32)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.repl = pl.repl_table()
        self.phat = torch.zeros(pl.p_elems, **f32)
        self.r = min(n, m, rank)

    def products(self, q):
        """p_w = M_w q for every worker (K1 with no EF add)."""
        pl, lib, sp = self.pl, _lib.lib(), stream_ptr()
        q_in = torch.zeros(pl.q_elems, **self.f32)
        pl.q_view(q_in, 0).copy_(q)
        ps = []
        for w in self.works:
            p = torch.zeros(pl.p_elems, **self.f32)
            _lib.check(lib.psgd_ef_p(pl.handle, ptr(w), None, ptr(self.scratch), ptr(q_in), ptr(p), None,
                                     ptr(self.status), sp), "psgd_ef_p")
            ps.append(p)
        return ps

    def mean(self, bufs, bits):
        """all_reduce_mean (comm.py:84-98): (buffer, divisor still to apply)."""
        if self.world == 1:
            return bufs[0], 1
        self.comm.charge_allreduce(bits)
        if self.dist:
            self.comm.all_reduce_sum_(bufs[0])
            return bufs[0], self.world
        out = torch.empty_like(bufs[0])
        tree_mean_(bufs, out)
        return out, 1

    def iterate(self, q):
        pl, lib, sp = self.pl, _lib.lib(), stream_ptr()
        pm, div = self.mean(self.products(q), FLOAT_BITS * self.n * self.r)
        qws = []
        for w in self.works:  # P-hat = MGS(P / div), q_w = M_w^T P-hat
            qw = torch.zeros(pl.q_elems, **self.f32)
            _lib.check(lib.psgd_q_ef(pl.handle, ptr(w), ptr(pm), div, ptr(self.repl), ptr(self.phat), ptr(qw),
                                     ptr(self.escratch), None, ptr(self.status), sp), "psgd_q_ef")
            qws.append(qw)
        qs = [q.clone() for q in qws] if self.dist else qws
        qbar, qdiv = self.mean(qs, FLOAT_BITS * self.m * self.r)
        if qdiv != 1:
            qbar = qbar / qdiv
        return qbar, qws

    def outer(self, p, q):
        """p q^T (K5), p in the P layout and q in the Q layout of the plan."""
        pl, lib, sp = self.pl, _lib.lib(), stream_ptr()
        out = torch.empty(pl.flat_elems, **self.f32)
        _lib.check(lib.psgd_decompress(pl.handle, ptr(p), ptr(q), 1, None, ptr(out), ptr(self.status), sp),
                   "psgd_decompress")
        return pl.matrix_view(out, 0).clone()

    def check(self):
        st = int(self.status.item())
        if st & (_lib.STATUS_NONFINITE_GRAD | _lib.STATUS_NONFINITE_P):
            raise ContractViolation("orthogonalize input contains non-finite entries")
        if st & _lib.STATUS_REPLACEMENT:
            raise RuntimeError(f"Gram-Schmidt needed more than {_lib.REPL_ATTEMPTS} replacement draws for a column")


class BestApproximation(Compressor):
    """Near-optimal rank-r reference: four fresh subspace iterations per call,
    no state reuse (compressors.py:400-438), on K1 / K2+K3 / K5."""

    name = "bestapprox"
    linear = True
    route = "allreduce"
    uses_error_feedback = True
    iterations = 4

    def __init__(self, rank=1, device=None):
        super().__init__(rank)
        self.device = device

    def round_trip(self, mats, ctx, comm):
        """compressors.py:407-420."""
        _check_mats(mats, comm)
        as_np = not isinstance(mats[0], torch.Tensor)
        dev = _device_of(mats, self.device)
        ds = [_to_dev(x, dev) for x in mats]
        n, m = ds[0].shape
        self._charge_compress(comm, n, m, len(ds))
        rank = min(n, m, self.rank)
        q = _to_dev(ctx.rng("fresh_start").standard_normal((m, rank)), dev)
        with torch.cuda.device(dev):
            R = _Rounds(ds, comm, self.rank, dev)
            for _ in range(self.iterations):
                qbar, qws = R.iterate(q)
                q = R.pl.q_view(qbar, 0).contiguous()
            comm.stats.decode_ops += 2 * n * m * rank
            agg = R.outer(R.phat, qbar)
            locs = [R.outer(R.phat, qw) for qw in qws]
            R.check()
        payload = LowRank(_out(R.pl.p_view(R.phat, 0).clone(), as_np), _out(q, as_np))
        return RoundTrip(_out(agg, as_np), [_out(x, as_np) for x in locs], payload)

    def compress(self, m, ctx):
        return self.round_trip([m], ctx, Communicator(1)).payload

    def payload_bits(self, n, m):
        return self.iterations * FLOAT_BITS * min(n, m, self.rank) * (n + m)

    def compress_cost(self, n, m):
        r = min(n, m, self.rank)
        return self.iterations * (4 * n * m * r + 2 * n * r * r + 3 * n * r)


class UnbiasedRankK(Compressor):
    """Rank-r sketch M u, u ~ N(0, 1/r) from the shared stream, never
    transmitted (compressors.py:444-468) with the reduce-route round trip
    (:255-269): the all-reduce averages proj; aggregate = mean(proj) u^T.
    K1 computes every proj, K5 every outer product."""

    name = "unbiased"
    linear = True
    route = "allreduce"
    uses_error_feedback = True

    def __init__(self, rank=1, device=None):
        super().__init__(rank)
        self.device = device

    def _u(self, ctx, n, m):
        rank = min(n, m, self.rank)
        return ctx.rng("projection").standard_normal((m, rank)) / np.sqrt(rank)

    def round_trip(self, mats, ctx, comm):
        _check_mats(mats, comm)
        as_np = not isinstance(mats[0], torch.Tensor)
        dev = _device_of(mats, self.device)
        ds = [_to_dev(x, dev) for x in mats]
        n, m = ds[0].shape
        self._charge_compress(comm, n, m, len(ds))
        u_host = self._u(ctx, n, m)
        u = _to_dev(u_host, dev)
        with torch.cuda.device(dev):
            R = _Rounds(ds, comm, self.rank, dev)
            ps = R.products(u)
            q_in = torch.zeros(R.pl.q_elems, **R.f32)
            R.pl.q_view(q_in, 0).copy_(u)
            locs = [R.outer(p, q_in) for p in ps]
            red, div = R.mean([p.clone() for p in ps] if R.dist else ps, self.payload_bits(n, m))
            if div != 1:
                red = red / div
            comm.stats.decode_ops += 2 * n * m * u.shape[1]
            agg = R.outer(red, q_in)
            R.check()
        proj = R.pl.p_view(red, 0).clone()
        payload = RandomProjection(_out(proj, as_np), u_host if as_np else u)
        return RoundTrip(_out(agg, as_np), [_out(x, as_np) for x in locs], payload)

    def compress(self, m, ctx):
        return self.round_trip([m], ctx, Communicator(1)).payload

    def payload_bits(self, n, m):
        return FLOAT_BITS * min(n, m, self.rank) * n

    def compress_cost(self, n, m):
        rank = min(n, m, self.rank)
        return 2 * n * m * rank + m * rank


COMPRESSORS = {PowerSGD.name: PowerSGD, BestApproximation.name: BestApproximation,
               UnbiasedRankK.name: UnbiasedRankK}


def make_compressor(name, rank=1):
    """compressors.py:703-707 (the low-rank family that runs on the B200 kernels:
    powersgd, bestapprox, unbiased)."""
    if name not in COMPRESSORS:
        raise ContractViolation(f"unknown compressor {name!r}; choose from {sorted(COMPRESSORS)}")
    return COMPRESSORS[name](rank=rank)

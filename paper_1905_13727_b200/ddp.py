"""PyTorch DDP communication hook backed by the B200 PowerSGD path.

Gradients arrive bucket by bucket during backward; each bucket is compressed as
soon as DDP hands it over, on a side stream, so compression and its exchanges
overlap the rest of backward (the reference packs one flat buffer after backward,
PAPER.md).  Per bucket, a
`PowerSGDEngine` over the bucket's parameters runs the reference's per-parameter
step (optimizer.py:110-129): delta = g + e, P = delta Q, all-reduce P (+ bias),
P-hat = MGS(P / W), q_w = delta^T P-hat, e = delta - P-hat q_w^T, all-reduce q,
M-hat = P-hat Q-bar^T.  The hook writes M-hat (the mean update) and the bias means
back into the bucket, so DDP's optimizer sees the aggregated gradient.  The
on-wire format is unchanged: packed P (+ bias) and packed q.

    state = PowerSGDState(model, rank=2, seed=0)
    ddp_model.register_comm_hook(state, powersgd_hook)

Warm-start Q is seeded per parameter from the model's parameter order, exactly as
the reference seeds it (derive_rng(seed, "warm_start_init", param_index)).
"""

import torch

from . import _lib
from .catalogs import ParamSpec
from .comm import DistributedCommunicator
from .engine import PowerSGDEngine


class PowerSGDState:
    """Hook state: one engine per bucket layout (created on its first call).  The
    error-feedback memory lives in the engines, so it follows a parameter only
    while its bucket layout is stable (DDP fixes the layout after iteration 1)."""

    def __init__(self, model, rank=2, seed=0, process_group=None, check_every=0):
        self.rank = int(rank)
        self.seed = int(seed)
        self.comm = DistributedCommunicator(process_group)
        self.param_index = {id(p): i for i, p in enumerate(model.parameters())}
        self.names = {id(p): n for n, p in model.named_parameters()}
        self.engines = {}
        self.owner = {}  # id(param) -> (engine, index in it): where its EF memory and Q live
        self.check_every = int(check_every)  # 0: never synchronise inside the hook
        self.calls = 0
        self.streams = {}  # device -> side stream the buckets' work runs on

    def stream_for(self, dev):
        s = self.streams.get(dev)
        if s is None:
            s = self.streams[dev] = torch.cuda.Stream(device=dev)
        return s

    @property
    def stats(self):
        return self.comm.stats

    @staticmethod
    def _pair(bucket):
        """(params, grads) in matching order (the two lists can come back in
        opposite orders on some torch versions)."""
        params, grads = list(bucket.parameters()), list(bucket.gradients())
        if len(params) == len(grads) and any(p.numel() != g.numel() for p, g in zip(params, grads)):
            params = params[::-1]
        if len(params) != len(grads) or any(p.numel() != g.numel() for p, g in zip(params, grads)):
            raise RuntimeError("cannot match the bucket's parameters to its gradients")
        return params, grads

    def engine_for(self, bucket):
        # keyed by the bucket's parameters: DDP rebuilds its buckets after the first
        # iteration, so an index can name different parameters over time
        params, _ = self._pair(bucket)
        key = tuple(id(p) for p in params)
        eng = self.engines.get(key)
        if eng is None:
            specs = [ParamSpec(self.names.get(id(p), f"p{self.param_index[id(p)]}"), tuple(p.shape))
                     for p in params]
            eng = PowerSGDEngine(specs, self.rank, comm=self.comm, seed=self.seed,
                                 device=params[0].device,
                                 param_indices=[self.param_index[id(p)] for p in params])
            for i, p in enumerate(params):  # a rebuilt bucket inherits e and the warm-start Q
                old = self.owner.get(id(p))
                if old is not None and not specs[i].is_bias:
                    oeng, oi = old
                    eng.error_view(i).copy_(oeng.error_view(oi))
                    eng.q_view(i).copy_(oeng.q_view(oi))
                self.owner[id(p)] = (eng, i)
            self.engines[key] = eng
            # engines of a superseded bucket layout own no parameter any more: free them
            live = {id(e) for e, _ in self.owner.values()}
            for k in [k for k, e in self.engines.items() if id(e) not in live]:
                del self.engines[k]
        return eng


def powersgd_hook(state, bucket):
    """DDP comm hook: compress, exchange and decompress one gradient bucket.

    The bucket's work (copies, kernels, the two all-reduces) is enqueued on a side
    stream that first waits for the backward stream, so it overlaps the rest of
    backward on the device; the hook never blocks the host.  The returned Future is
    CUDA-aware: DDP's use of the result waits for the side stream."""
    eng = state.engine_for(bucket)
    _, grads = state._pair(bucket)
    dev = eng.device
    cur = torch.cuda.current_stream(dev)
    side = state.stream_for(dev)
    side.wait_stream(cur)
    with torch.cuda.stream(side):
        for i, g in enumerate(grads):
            eng.grad_view(i).copy_(g.view(eng.specs[i].shape))
        eng.run(side)
        for i, g in enumerate(grads):
            g.copy_(eng.update_view(i).reshape(g.shape))
        # A non-finite gradient on any rank (the flags ride in the P all-reduce, so every
        # rank's status agrees) leaves e and Q untouched but no M-hat: poison the whole
        # bucket on every rank, so an AMP GradScaler skips the step everywhere instead of
        # the replicas applying different updates (the reference raises on all workers).
        bad = (eng.status & (_lib.STATUS_NONFINITE_GRAD | _lib.STATUS_NONFINITE_P)) != 0
        bucket.buffer().masked_fill_(bad, float("nan"))
        state.calls += 1
        if state.check_every and state.calls % state.check_every == 0:
            eng.check()
        fut = torch.futures.Future(devices=[dev])
        fut.set_result(bucket.buffer())
    return fut

"""The grouped PowerSGD step: every parameter of a model in one kernel sequence.

This is the fast path behind the reference's per-parameter loop
(optimizer.py:110-129, compressors.py:369-379).  One `PowerSGDEngine` owns,
on one device, the packed fp32 buffers of a parameter catalog:

    g[w]      flat gradients of local worker w       (caller fills; `grad_view`)
    e[w]      error-feedback memory                  (WorkerState.error, optimizer.py:63)
    work[w]   delta, then M-hat                      (RoundTrip.aggregated)
    P[w]      packed P + bias tail + non-finite flags (AR1 payload)
    Phat      P-hat of every matrix                  (RoundTrip.payload.p)
    Q         warm-start Q of every matrix           (PowerSGD.q_memory, compressors.py:357)
    qbuf[w]   local q_w                              (AR2 payload, W > 1)
    bias_out  mean of the bias gradients             (optimizer.py:111-113)

and runs, per step,

    W == 1 (one GPU)        psgd_step_single                       (K1, K2, K3)
    W > 1, distributed      K1 | all_reduce(P) | K2, K3 | all_reduce(q) | K5
    W > 1, simulated        K1 x W | tree_mean | K2, K3 x W | tree_mean | K5

Every mode can be captured into one CUDA graph (`capture()`), the NCCL
all-reduces of the distributed mode included.

Q is seeded exactly as the reference (derive_rng(seed, "warm_start_init",
param_index), compressors.py:362-367) and CommStats are charged exactly as the
reference charges them (compressors.py:248-249, 374; comm.py:96).
"""

import ctypes

import torch

from . import _lib
from .comm import CommStats, tree_mean_
from .distributed import first_nonfinite_site, step_charges
from .linalg import ContractViolation
from .plan import Plan, ptr, stream_ptr
from .seeding import warm_start_q


class NonFiniteGradient(RuntimeError):
    """optimizer.py:31-38: a worker produced a NaN/inf gradient; names the site."""

    def __init__(self, param_name, worker):
        super().__init__(f"non-finite gradient for parameter {param_name!r} on worker {worker}")
        self.param_name = param_name
        self.worker = worker


class PowerSGDEngine:
    """Grouped, warm-started, error-feedback PowerSGD over a parameter catalog.

    specs:   ParamSpec list in catalog order (param_index = position, biases included).
    rank:    requested rank r; each matrix uses min(n, m, r) (compressors.py:359-360).
    workers: simulated workers on this device (the reference's W-list model);
             must be 1 when `comm` is a DistributedCommunicator.
    comm:    Communicator / DistributedCommunicator whose CommStats are charged.
    exchange: run the W > 1 exchange sequence (K1, all-reduce P, K2/K3,
             all-reduce q, K5) even when the distributed group has one rank, so the
             collectives are issued (tests the NCCL path on a single GPU).
    """

    def __init__(self, specs, rank, *, workers=1, comm=None, seed=0, device=None,
                 error_feedback=True, param_indices=None, exchange=False):
        self.specs = list(specs)
        # the reference's param_index (seeds the warm start): catalog position, or the
        # caller's global indices when the specs are a subset (e.g. one DDP bucket)
        self.param_indices = list(range(len(self.specs))) if param_indices is None else list(param_indices)
        if len(self.param_indices) != len(self.specs):
            raise ValueError("param_indices must match specs")
        self.rank = int(rank)
        if self.rank < 1:
            raise ContractViolation(f"rank must be >= 1, got {rank}")
        self.distributed = bool(comm is not None and getattr(comm, "distributed", False))
        if self.distributed and workers != 1:
            raise ValueError("a distributed worker owns exactly one local gradient set")
        if comm is not None and not self.distributed and comm.world_size != workers:
            raise ValueError(f"expected {comm.world_size} workers, got {workers}")
        self.world = comm.world_size if self.distributed else int(workers)
        self.nlocal = 1 if self.distributed else int(workers)
        if exchange and not self.distributed:
            raise ValueError("exchange=True needs a DistributedCommunicator")
        self.exchange = bool(exchange) or self.world > 1
        self.plan_world = max(2, self.world) if self.exchange else 1
        self.comm = comm
        self.stats = comm.stats if comm is not None else CommStats()
        self.seed = int(seed)
        self.error_feedback = bool(error_feedback)

        self.mat_index = [i for i, s in enumerate(self.specs) if not s.is_bias]
        self.bias_index = [i for i, s in enumerate(self.specs) if s.is_bias]
        self.slot = {pi: k for k, pi in enumerate(self.mat_index)}
        self.bias_off = {}
        off = 0
        for pi in self.bias_index:
            self.bias_off[pi] = off
            off += self.specs[pi].size
        self.nbias = off

        shapes = [self.specs[pi].matrix_shape for pi in self.mat_index]
        self.plan = Plan(shapes, self.rank, self.plan_world, self.nbias, device)
        dev = self.device = self.plan.device
        pl = self.plan
        z = dict(dtype=torch.float32, device=dev)
        L = self.nlocal
        self.g = [torch.zeros(pl.flat_elems, **z) for _ in range(L)]
        self.e = [torch.zeros(pl.flat_elems, **z) for _ in range(L)]
        self.work = [torch.zeros(pl.flat_elems, **z) for _ in range(L)]
        self.bias_g = [torch.zeros(max(1, self.nbias), **z) for _ in range(L)]
        self.P = [torch.zeros(pl.p_elems, **z) for _ in range(L)]
        self.Pm = torch.zeros(pl.p_elems, **z) if L > 1 else self.P[0]
        self.Phat = torch.zeros(pl.p_elems, **z)
        self.Q = torch.zeros(pl.q_elems, **z)
        self.qbuf = [torch.zeros(pl.q_elems, **z) for _ in range(L)] if self.exchange else None
        self.bias_out = torch.zeros(max(1, self.nbias), **z)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        # EF off: the EF output of K3 lands in a scratch buffer nobody reads
        self._e_scratch = None if self.error_feedback else torch.empty(pl.flat_elems, **z)
        self.repl = pl.repl_table()
        for k, pi in enumerate(self.mat_index):
            mi = pl.matrices[k]
            q0 = warm_start_q(self.seed, self.param_indices[pi], mi.m, mi.r_eff)
            pl.q_view(self.Q, k).copy_(torch.from_numpy(q0))
        self.step_count = 0
        self._graph = None
        self.fused = self._fused_ok = False
        # host-side accounting per step (integers), charged as the reference does
        self._charge = step_charges([(mi.n, mi.m, mi.r_eff) for mi in pl.matrices], self.nbias, self.world)

    # ------------------------------------------------------------------ views
    def grad_view(self, param_index, worker=0):
        """Where worker `worker` puts the gradient of parameter `param_index` (spec shape)."""
        s = self.specs[param_index]
        if s.is_bias:
            o = self.bias_off[param_index]
            return self.bias_g[worker][o:o + s.size]
        return self.plan.matrix_view(self.g[worker], self.slot[param_index]).view(s.shape)

    def update_view(self, param_index):
        """Aggregated update of `param_index` after a step: M-hat or the bias mean."""
        s = self.specs[param_index]
        if s.is_bias:
            o = self.bias_off[param_index]
            return self.bias_out[o:o + s.size]
        return self.plan.matrix_view(self.work[0], self.slot[param_index]).view(s.shape)

    def error_view(self, param_index, worker=0):
        return self.plan.matrix_view(self.e[worker], self.slot[param_index])

    def p_view(self, param_index):
        """P-hat of `param_index` after a step (RoundTrip.payload.p)."""
        return self.plan.p_view(self.Phat, self.slot[param_index])

    def q_view(self, param_index):
        """Warm-start Q of `param_index` (= Q-bar of the last step, payload.q)."""
        return self.plan.q_view(self.Q, self.slot[param_index])

    def local_q_view(self, param_index, worker=0):
        if self.qbuf is None:
            return self.q_view(param_index)
        return self.plan.q_view(self.qbuf[worker], self.slot[param_index])

    # ------------------------------------------------------------------ the step
    def _enqueue(self, stream=None):
        lib = _lib.lib()
        pl = self.plan
        sp = stream_ptr(stream)
        h = pl.handle
        e = self.e if self.error_feedback else [self._e_scratch] * self.nlocal
        ein = self.e if self.error_feedback else [None] * self.nlocal
        sgd = self._sgd_struct() if self._fused_ok else None
        if not self.exchange and self.error_feedback:
            if sgd is not None:  # K3 applies the heavy-ball update from the M-hat registers
                _lib.check(lib.psgd_step_single_sgd(
                    h, ptr(self.g[0]), ptr(e[0]), ptr(self.work[0]), ptr(self.Q), ptr(self.P[0]), ptr(self.Phat),
                    ptr(self.bias_g[0]), ptr(self.repl), ptr(self.bias_out), ctypes.byref(sgd), ptr(self.status),
                    sp), "psgd_step_single_sgd")
                return
            _lib.check(lib.psgd_step_single(h, ptr(self.g[0]), ptr(e[0]), ptr(self.work[0]), ptr(self.Q),
                                            ptr(self.P[0]), ptr(self.Phat), ptr(self.bias_g[0]), ptr(self.repl),
                                            ptr(self.bias_out), ptr(self.status), sp), "psgd_step_single")
            self._unfused_update(sp)
            return
        for w in range(self.nlocal):      # K1: delta = g + e, P = delta Q  (e NULL: EF off)
            _lib.check(lib.psgd_ef_p(h, ptr(self.g[w]), ptr(ein[w]), ptr(self.work[w]), ptr(self.Q),
                                     ptr(self.P[w]), ptr(self.bias_g[w]), ptr(self.status), sp), "psgd_ef_p")
        if self.distributed:              # AR1 (P + bias + flags), / W fused into K2
            self.comm.all_reduce_sum_(self.P[0], force=self.exchange)
            div = self.world
        elif self.nlocal > 1:
            tree_mean_(self.P, self.Pm, stream)
            div = 1
        else:
            div = 1
        for w in range(self.nlocal):      # K2 + K3: GS, q_w, e (+ M-hat and Q when there is no exchange)
            q_w = self.qbuf[w] if self.exchange else self.Q
            _lib.check(lib.psgd_q_ef(h, ptr(self.work[w]), ptr(self.Pm), div, ptr(self.repl), ptr(self.Phat),
                                     ptr(q_w), ptr(e[w]), ptr(self.bias_out), ptr(self.status), sp), "psgd_q_ef")
        if not self.exchange:
            self._unfused_update(sp)
            return
        if self.distributed:              # AR2 (q), then Q-bar = q / W and M-hat
            self.comm.all_reduce_sum_(self.qbuf[0], force=True)
            qs, div, qstore = self.qbuf[0], self.world, self.Q
        else:
            tree_mean_(self.qbuf, self.Q, stream)
            qs, div, qstore = self.Q, 1, None
        if sgd is not None:               # K5 applies the heavy-ball update from the M-hat registers
            _lib.check(lib.psgd_decompress_sgd(h, ptr(self.Phat), ptr(qs), div, ptr(qstore), ptr(self.work[0]),
                                               ptr(self.bias_out), ctypes.byref(sgd), ptr(self.status), sp),
                       "psgd_decompress_sgd")
            return
        _lib.check(lib.psgd_decompress(h, ptr(self.Phat), ptr(qs), div, ptr(qstore), ptr(self.work[0]),
                                       ptr(self.status), sp), "psgd_decompress")
        self._unfused_update(sp)

    def _scratch_e(self):
        return self._e_scratch

    # ------------------------------------------------------------------ optimizer (optimizer.py:131-134)
    def attach_optimizer(self, lr, momentum, params=None, fused=False, keep_update=True):
        """Heavy-ball state on the device, in the plan's packed layout: parameters
        x and momentum buffers m (Optimizer.params / momentum_buffers,
        optimizer.py:47-55).  `params`: initial values in catalog order.

        fused=True: every later step applies the update itself, like the
        reference's optimizer.step (optimizer.py:98-135) — inside the kernel that
        produces M-hat (K3 at W = 1, K5 at W > 1), consuming M-hat from registers,
        when the plan allows it (`fused_in_kernel`), else with the one-pass update
        kernel appended to the step; `optimizer_step()` is then a no-op.
        keep_update=False (fused only): M-hat is not stored (update_view is stale)."""
        z = dict(dtype=torch.float32, device=self.device)
        self.lr, self.momentum = float(lr), float(momentum)
        self.fused = bool(fused)
        self.keep_update = bool(keep_update) or not self.fused
        self._fused_ok = self.fused and bool(self.plan.info.opt_fusable) and (self.exchange or self.error_feedback)
        self._graph = None  # a captured step no longer matches
        self.params = torch.zeros(self.plan.flat_elems, **z)
        self.mom = torch.zeros(self.plan.flat_elems, **z)
        self.bias_params = torch.zeros(max(1, self.nbias), **z)
        self.bias_mom = torch.zeros(max(1, self.nbias), **z)
        if params is not None:
            for i, p in enumerate(params):
                self.param_view(i).copy_(torch.as_tensor(p, dtype=torch.float32).reshape(self.specs[i].shape))

    def _flat_view(self, flat, bias_flat, param_index):
        s = self.specs[param_index]
        if s.is_bias:
            o = self.bias_off[param_index]
            return bias_flat[o:o + s.size]
        return self.plan.matrix_view(flat, self.slot[param_index]).view(s.shape)

    def param_view(self, param_index):
        return self._flat_view(self.params, self.bias_params, param_index)

    def momentum_view(self, param_index):
        return self._flat_view(self.mom, self.bias_mom, param_index)

    @property
    def fused_in_kernel(self):
        """The attached optimizer runs inside K3 / K5 (not as a separate pass)."""
        return self._fused_ok

    def _sgd_struct(self):
        return _lib.Sgd(self.params.data_ptr(), self.mom.data_ptr(), self.bias_params.data_ptr(),
                        self.bias_mom.data_ptr(), self.lr, self.momentum, 1 if self.keep_update else 0, 0)

    def _unfused_update(self, sp):
        if self.fused and not self._fused_ok:
            self._momentum_launch(sp)

    def optimizer_step(self, stream=None):
        """m = momentum m + u ; x -= lr (u + m) for every parameter, one kernel,
        with u = the aggregated update of the last step (M-hat, bias mean).
        A no-op when the optimizer is fused into the step (attach_optimizer(fused=True))."""
        if self.fused:
            return
        self._momentum_launch(stream_ptr(stream))

    def _momentum_launch(self, sp):
        _lib.check(_lib.lib().psgd_momentum_step(
            self.plan.handle, ptr(self.params), ptr(self.mom), ptr(self.work[0]), ptr(self.bias_params),
            ptr(self.bias_mom), ptr(self.bias_out), self.lr, self.momentum, ptr(self.status),
            sp), "psgd_momentum_step")

    def run(self, stream=None):
        """Enqueue one step on `stream` (default: current) without synchronising."""
        self._run_device(stream)
        self._account()

    def _run_device(self, stream=None):
        if self._graph is not None:
            if stream is not None:
                with torch.cuda.stream(stream):
                    self._graph.replay()
            else:
                self._graph.replay()
        else:
            self._enqueue(stream)

    def _account(self):
        """CommStats of one step, charged as the reference charges them."""
        b, f, d = self._charge
        self.stats.bits_allreduced += b
        self.stats.compress_flops += f
        self.stats.decode_ops += d
        self.step_count += 1

    def step(self, check=True):
        self.run()
        if check:
            self.check()

    def capture(self):
        """Capture the step into a CUDA graph; later `run`s replay it.  In the
        distributed mode the two NCCL all-reduces are captured with the kernels
        (the communicator is initialised by a warm-up collective first)."""
        if self.distributed:
            warm = torch.zeros(1, dtype=torch.float32, device=self.device)
            self.comm.all_reduce_sum_(warm, force=True)
            torch.cuda.synchronize(self.device)
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                self._enqueue(s)
        torch.cuda.current_stream(self.device).wait_stream(s)
        self._graph = g
        return g

    # ------------------------------------------------------------------ errors
    def check(self):
        """Synchronise on the status word and raise what the reference would."""
        st = int(self.status.item())
        if self.distributed:
            import torch.distributed as dist
            t = torch.tensor([st], dtype=torch.int32, device=self.device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.comm.group)
            st = int(t.item())
        if st == 0:
            return
        if st & (_lib.STATUS_NONFINITE_GRAD | _lib.STATUS_NONFINITE_P):
            site = self._first_nonfinite()
            if site is not None:
                raise NonFiniteGradient(*site)
            raise ContractViolation("orthogonalize input contains non-finite entries")
        if st & _lib.STATUS_REPLACEMENT:
            raise RuntimeError(f"Gram-Schmidt needed more than {_lib.REPL_ATTEMPTS} replacement draws for a column")

    def _first_nonfinite(self):
        """(param name, worker) of the first non-finite gradient, worker-major as
        optimizer.py:72-76 scans.  Error path only."""
        local = None
        for w in range(self.nlocal):
            for pi, s in enumerate(self.specs):
                if not bool(torch.isfinite(self.grad_view(pi, w)).all()):
                    local = (w, pi)
                    break
            if local is not None:
                break
        if not self.distributed:
            return None if local is None else (self.specs[local[1]].name, local[0])
        site = first_nonfinite_site(None if local is None else local[1], self.comm, len(self.specs))
        return None if site is None else (self.specs[site[0]].name, site[1])

"""Host gradients in, host update out, with the PCIe transfers overlapped.

`HostPipelinedEngine` is the W = 1 step for gradients that live in (pinned) host
memory, e.g. produced on the CPU or staged by a data pipeline: the catalog is cut
into parameter groups, each with its own `PowerSGDEngine` (param_index = catalog
position, so the warm start is seeded exactly as the reference seeds it), and per
group the host->device copy, the compression step (optimizer.py:110-129) and the
device->host copy of M-hat / the bias mean run on three streams:

    h2d:      g_0 | g_1 | g_2 | ... | g_G-1
    compute:        step_0 | step_1 | ...   | step_G-1
    d2h:                   M_0    | M_1 ... |          M_G-1

so the copies of one group overlap the other groups' compression and the two PCIe
directions overlap each other.  The step time is then about the bidirectional
transfer time plus the first group's H2D and the last group's D2H, so the first
and the last group are small (the catalog's smallest parameters) and the rest are
balanced.  The whole multi-stream step (copies, kernels, cross-stream
dependencies) is captured into one CUDA graph: replaying it avoids the tens of
microseconds an eager cross-stream event hand-off costs per group.  Results are
identical to one engine over the whole catalog (the reference's per-parameter loop
is independent across parameters).
"""

import os

import torch

from .engine import PowerSGDEngine


def split_groups(specs, groups):
    """Contiguous parameter groups of ~equal element count (catalog order)."""
    total = sum(s.size for s in specs) or 1
    out, cur, acc = [], [], 0
    for i, s in enumerate(specs):
        cur.append(i)
        acc += s.size
        if acc >= total * (len(out) + 1) / groups and len(out) < groups - 1:
            out.append(cur)
            cur = []
    if cur:
        out.append(cur)
    return [g for g in out if g]


def transfer_groups(specs, groups, edge=0.02, edge_groups=1):
    """Groups in transfer order for the pipelined step: `edge_groups` small groups
    first (the smallest parameters, ~`edge` of the bytes each, so compression and the
    device->host stream start early), `edge_groups` small groups last (the next
    smallest, so the final device->host copies are short), and the remaining
    parameters in catalog order cut into `groups - 2 edge_groups` groups of ~equal
    size.  Every parameter appears exactly once; each group lists its parameters in
    catalog order."""
    n = len(specs)
    ne = max(1, int(edge_groups))
    if groups < 2 * ne + 1 or n < 2 * ne + 1:
        return split_groups(specs, max(1, groups))
    total = sum(s.size for s in specs) or 1
    order = iter(sorted(range(n), key=lambda i: (specs[i].size, i)))
    edges = []
    for _ in range(2 * ne):
        cur, acc = [], 0
        for i in order:
            cur.append(i)
            acc += specs[i].size
            if acc >= edge * total:
                break
        if cur:
            edges.append(sorted(cur))
    taken = {i for g in edges for i in g}
    rest = [i for i in range(n) if i not in taken]
    middle = []
    if rest:
        sub = split_groups([specs[i] for i in rest], max(1, groups - 2 * ne))
        middle = [[rest[j] for j in g] for g in sub]
    first, last = edges[0::2], edges[1::2][::-1]  # the smallest at the very start and the very end
    return [g for g in first + middle + last if g]


class HostPipelinedEngine:
    """graphs: "step" (default) captures the whole pipelined step into one CUDA
    graph; "engine" captures each group's compression only (cross-stream hand-offs
    eager); False runs everything eagerly."""

    def __init__(self, specs, rank, *, groups=10, seed=0, device=None, graphs="step", order="transfer",
                 edge_groups=None):
        self.specs = list(specs)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if edge_groups is None:
            edge_groups = int(os.environ.get("PSGD_E2E_EDGE", "1"))
        self.groups = (transfer_groups(self.specs, groups, edge_groups=edge_groups) if order == "transfer"
                       else split_groups(self.specs, groups))
        self.engines = [PowerSGDEngine([self.specs[i] for i in g], rank, seed=seed, device=self.device,
                                       param_indices=g) for g in self.groups]
        self.where = {pi: (k, j) for k, g in enumerate(self.groups) for j, pi in enumerate(g)}
        pin = dict(dtype=torch.float32, pin_memory=True)
        self.g_host = [torch.zeros(e.g[0].numel(), **pin) for e in self.engines]
        self.bias_host = [torch.zeros(e.bias_g[0].numel(), **pin) for e in self.engines]
        self.out_host = [torch.zeros(e.work[0].numel(), **pin) for e in self.engines]
        self.bias_out_host = [torch.zeros(e.bias_out.numel(), **pin) for e in self.engines]
        self.s_h2d = torch.cuda.Stream(device=self.device)
        self.s_cmp = torch.cuda.Stream(device=self.device)
        self.s_d2h = torch.cuda.Stream(device=self.device)
        self._graph = None
        if graphs == "engine" or graphs is True:
            for e in self.engines:
                e.capture()
        elif graphs == "step":
            self._capture()

    # host views in the spec shapes (the engines' packed layouts, pinned)
    def _host(self, flat, bias, k, j):
        e = self.engines[k]
        pi = self.groups[k][j]
        s = self.specs[pi]
        if s.is_bias:
            o = e.bias_off[j]
            return bias[k][o:o + s.size].view(s.shape)
        return e.plan.matrix_view(flat[k], e.slot[j]).view(s.shape)

    def grad_host_view(self, param_index):
        return self._host(self.g_host, self.bias_host, *self.where[param_index])

    def update_host_view(self, param_index):
        return self._host(self.out_host, self.bias_out_host, *self.where[param_index])

    def error_view(self, param_index):
        k, j = self.where[param_index]
        return self.engines[k].error_view(j)

    @property
    def h2d_bytes(self):
        return 4 * sum(t.numel() for t in self.g_host + self.bias_host)

    @property
    def d2h_bytes(self):
        return 4 * sum(t.numel() for t in self.out_host + self.bias_out_host)

    def _enqueue(self, origin, raw):
        """The pipelined step after `origin`'s work; `origin` waits for its end.
        raw: launch the compression kernels directly (inside a graph capture)."""
        for s in (self.s_h2d, self.s_cmp, self.s_d2h):
            s.wait_stream(origin)
        done_in, done_cmp = [], []
        with torch.cuda.stream(self.s_h2d):
            for k, e in enumerate(self.engines):
                e.g[0].copy_(self.g_host[k], non_blocking=True)
                if e.nbias:
                    e.bias_g[0].copy_(self.bias_host[k], non_blocking=True)
                done_in.append(torch.cuda.Event())
                done_in[-1].record(self.s_h2d)
        with torch.cuda.stream(self.s_cmp):
            for k, e in enumerate(self.engines):
                self.s_cmp.wait_event(done_in[k])
                if raw:
                    e._enqueue(self.s_cmp)
                else:
                    e._run_device(self.s_cmp)
                done_cmp.append(torch.cuda.Event())
                done_cmp[-1].record(self.s_cmp)
        with torch.cuda.stream(self.s_d2h):
            for k, e in enumerate(self.engines):
                self.s_d2h.wait_event(done_cmp[k])
                self.out_host[k].copy_(e.work[0], non_blocking=True)
                if e.nbias:
                    self.bias_out_host[k].copy_(e.bias_out, non_blocking=True)
        origin.wait_stream(self.s_d2h)
        origin.wait_stream(self.s_cmp)

    def _capture(self):
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                self._enqueue(s, raw=True)
        torch.cuda.current_stream(self.device).wait_stream(s)
        self._graph = g

    def step(self):
        """Enqueue one step (transfers + compression) after the current stream's work;
        the current stream waits for the last device->host copy."""
        if self._graph is not None:
            self._graph.replay()
        else:
            self._enqueue(torch.cuda.current_stream(self.device), raw=False)
        for e in self.engines:
            e._account()

    def check(self):
        for e in self.engines:
            e.check()

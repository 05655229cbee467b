"""Host gradients in, host update out, with the PCIe transfers overlapped.

`HostPipelinedEngine` is the W = 1 step for gradients that live in (pinned) host
memory, e.g. produced on the CPU or staged by a data pipeline: the catalog is cut
into parameter groups, each with its own `PowerSGDEngine` (param_index = catalog
position, so the warm start is seeded exactly as the reference seeds it), and per
group the host->device copy, the compression step (optimizer.py:110-129) and the
device->host copy of M-hat / the bias mean run on three streams:

    h2d:      g_0 | g_1 | g_2 | g_3
    compute:        step_0 | step_1 | step_2 | step_3
    d2h:                   M_0    | M_1    | M_2    | M_3

so the copies of one group overlap the other groups' compression and the two PCIe
directions overlap each other.  Results are identical to one engine over the whole
catalog (the reference's per-parameter loop is independent across parameters).
"""

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


class HostPipelinedEngine:
    def __init__(self, specs, rank, *, groups=4, seed=0, device=None, graphs=True):
        self.specs = list(specs)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.groups = split_groups(self.specs, groups)
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
        if graphs:
            for e in self.engines:
                e.capture()

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

    def step(self):
        """Enqueue one step (transfers + compression) after the current stream's work;
        the current stream waits for the last device->host copy."""
        cur = torch.cuda.current_stream(self.device)
        for s in (self.s_h2d, self.s_cmp, self.s_d2h):
            s.wait_stream(cur)
        done_in, done_cmp = [], []
        with torch.cuda.stream(self.s_h2d):
            for k, e in enumerate(self.engines):
                e.g[0].copy_(self.g_host[k], non_blocking=True)
                e.bias_g[0].copy_(self.bias_host[k], non_blocking=True)
                done_in.append(torch.cuda.Event())
                done_in[-1].record(self.s_h2d)
        with torch.cuda.stream(self.s_cmp):
            for k, e in enumerate(self.engines):
                self.s_cmp.wait_event(done_in[k])
                e.run(self.s_cmp)
                done_cmp.append(torch.cuda.Event())
                done_cmp[-1].record(self.s_cmp)
        with torch.cuda.stream(self.s_d2h):
            for k, e in enumerate(self.engines):
                self.s_d2h.wait_event(done_cmp[k])
                self.out_host[k].copy_(e.work[0], non_blocking=True)
                self.bias_out_host[k].copy_(e.bias_out, non_blocking=True)
        cur.wait_stream(self.s_d2h)
        cur.wait_stream(self.s_cmp)

    def check(self):
        for e in self.engines:
            e.check()

"""Does splitting the step into matrix groups (K1->K2->K3 per group, so each group's
delta is still in L2 when its K3 reads it) beat one pass?  GPU box only."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_13727_b200 import PowerSGDEngine, catalogs  # noqa: E402

specs = list(catalogs.RESNET18.params)
mats = [i for i, s in enumerate(specs) if not s.is_bias]
total = sum(specs[i].size for i in mats)
flush = torch.empty(64 << 20, device="cuda")


def split(k):
    groups, cur, acc = [], [], 0
    for i, s in enumerate(specs):
        cur.append(s)
        acc += s.size if not s.is_bias else 0
        if acc >= total * (len(groups) + 1) / k and len(groups) < k - 1:
            groups.append(cur)
            cur = []
    groups.append(cur)
    return [g for g in groups if g]


for k in (1, 2, 3, 4):
    engs = [PowerSGDEngine(g, 2, seed=0) for g in split(k)]
    for e in engs:
        e.g[0].normal_()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        for e in engs:
            e._enqueue(s)
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=s):
            for e in engs:
                e._enqueue(s)
    torch.cuda.current_stream().wait_stream(s)
    ts = []
    for it in range(40):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        graph.replay()
        b.record()
        torch.cuda.synchronize()
        if it >= 5:
            ts.append(a.elapsed_time(b) * 1e3)
    print(f"groups {k}: sizes {[sum(p.size for p in g if not p.is_bias) for g in split(k)]} "
          f"step median {statistics.median(ts):.2f} us")

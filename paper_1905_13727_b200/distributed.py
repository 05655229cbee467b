"""Host-side logic of the one-worker-per-GPU exchange (kept free of CUDA so it
is testable with gloo on CPU; tests/test_distributed_cpu.py).

Per step each rank all-reduces (sum) two packed buffers: P ⊕ bias ⊕
non-finite flags (AR1, compressors.py:337 + optimizer.py:111-113) and q
(AR2, compressors.py:340); the ÷W of comm.py:97-98 is fused into the next
kernel.  CommStats are charged as the reference charges them.
"""

import torch


def step_charges(mats, nbias, world):
    """(bits_allreduced, compress_flops, decode_ops) of one step, as the reference's
    optimizer.step charges them: per matrix compress_flops += W * compress_cost
    (compressors.py:248-249, 389-391), decode_ops += 2 n m r (:374, :176-182), and for
    W > 1 bits += 32 n r + 32 m r (:337, :340 via comm.py:96) plus 32 per bias scalar
    (optimizer.py:111-113).  `mats`: iterable of (n, m, r_eff)."""
    bits = flops = dec = 0
    for n, m, r in mats:
        flops += world * (4 * n * m * r + 2 * n * r * r + 3 * n * r)
        dec += 2 * n * m * r
        if world > 1:
            bits += 32 * n * r + 32 * m * r
    if world > 1:
        bits += 32 * nbias
    return bits, flops, dec


def reduce_packed_(buf, comm):
    """AR1 / AR2: in-place sum over the workers (NCCL on GPUs, gloo in tests)."""
    return comm.all_reduce_sum_(buf)


def first_nonfinite_site(local_param, comm, nparams):
    """(param_index, worker) of the first non-finite gradient in the reference's
    worker-major scan order (optimizer.py:72-76), given this rank's first bad
    param index (or None).  Collective: every rank must call it."""
    import torch.distributed as dist
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(comm.group) == "nccl" \
        else torch.device("cpu")
    big = nparams + 1
    mine = torch.tensor([big if local_param is None else int(local_param)], dtype=torch.int64, device=dev)
    allv = [torch.zeros_like(mine) for _ in range(comm.world_size)]
    dist.all_gather(allv, mine, group=comm.group)
    for rank, v in enumerate(allv):
        if int(v.item()) < big:
            return int(v.item()), rank
    return None

"""Collectives of the hot path: the reference's simulated W-worker all-reduce
(comm.py:70-98) on one device, and the real thing over NCCL.

* `Communicator(W)` — the reference's own model: W workers as list entries in
  one process.  Device tensors are reduced by the `psgd_tree_mean` kernel in
  the reference's pairing order ((v0+v1)+(v2+v3))+..., then / W (comm.py:51-67,
  97-98); W == 1 is a free copy that charges nothing (comm.py:92-93).
* `DistributedCommunicator(group)` — one process per GPU = one worker.  The
  packed P / q buffers are summed in place with `torch.distributed.all_reduce`
  (NCCL over NVLink); the / W is fused into the next kernel.

Both charge `CommStats` exactly as the reference does (comm.py:23-48, 96).
"""

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from .plan import ptr, stream_ptr


@dataclass
class CommStats:
    bits_allreduced: int = 0
    bits_gathered: int = 0
    decode_ops: int = 0
    compress_flops: int = 0

    @property
    def bits_transmitted(self):
        return self.bits_allreduced + self.bits_gathered

    def snapshot(self):
        return CommStats(self.bits_allreduced, self.bits_gathered, self.decode_ops,
                         self.compress_flops)

    def since(self, earlier):
        return CommStats(self.bits_allreduced - earlier.bits_allreduced,
                         self.bits_gathered - earlier.bits_gathered,
                         self.decode_ops - earlier.decode_ops,
                         self.compress_flops - earlier.compress_flops)


def tree_mean_(bufs, out, stream=None):
    """out = tree_sum(bufs) / len(bufs) on the device (psgd_tree_mean)."""
    n = len(bufs)
    if n < 1 or n > _lib.MAX_TREE:
        raise ValueError(f"tree mean over {n} buffers (1..{_lib.MAX_TREE})")
    count = out.numel()
    for b in bufs:
        if b.numel() < count or b.dtype != torch.float32 or not b.is_cuda:
            raise ValueError("tree mean buffers must be fp32 CUDA tensors covering `out`")
    arr = (ctypes.c_void_p * n)(*[b.data_ptr() for b in bufs])
    _lib.check(_lib.lib().psgd_tree_mean(arr, n, count, ptr(out), stream_ptr(stream)),
               "psgd_tree_mean")
    return out


class Communicator:
    """Simulated collectives over `world_size` workers living on one device."""

    distributed = False

    def __init__(self, world_size, stats=None):
        if world_size < 1:
            raise ValueError(f"world_size must be >= 1, got {world_size}")
        self.world_size = world_size
        self.stats = stats if stats is not None else CommStats()

    def _check(self, per_worker):
        if len(per_worker) != self.world_size:
            raise ValueError(f"expected {self.world_size} entries, got {len(per_worker)}")

    def charge_allreduce(self, payload_bits):
        if self.world_size > 1:
            self.stats.bits_allreduced += payload_bits

    def all_reduce_mean(self, arrays, payload_bits=None):
        """comm.py:84-98 on the device.  numpy in -> float64 numpy out."""
        import numpy as np
        self._check(arrays)
        is_np = not isinstance(arrays[0], torch.Tensor)
        ts = [torch.as_tensor(np.asarray(a, dtype=np.float32)).cuda() if is_np
              else a.detach().float().contiguous() for a in arrays]
        if self.world_size == 1:
            out = ts[0].clone()
        else:
            self.stats.bits_allreduced += 32 * ts[0].numel() if payload_bits is None else payload_bits
            out = torch.empty_like(ts[0])
            tree_mean_([t.view(-1) for t in ts], out.view(-1))
        return out.double().cpu().numpy() if is_np else out

    def all_gather(self, payloads, payload_bits):
        """comm.py:100-104 (gather-route compressors; bookkeeping only)."""
        self._check(payloads)
        self.stats.bits_gathered += self.world_size * payload_bits
        return list(payloads)


class DistributedCommunicator:
    """One worker per process/GPU; sums over NCCL."""

    distributed = True

    def __init__(self, group=None, stats=None):
        import torch.distributed as dist
        if not dist.is_initialized():
            raise RuntimeError("torch.distributed is not initialised")
        self.group = group
        self.world_size = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.stats = stats if stats is not None else CommStats()

    def charge_allreduce(self, payload_bits):
        if self.world_size > 1:
            self.stats.bits_allreduced += payload_bits

    def all_reduce_sum_(self, t, force=False):
        """In-place sum over the ranks; `force` issues the collective even for a
        one-rank group (exercises the NCCL path on a single GPU)."""
        import torch.distributed as dist
        if self.world_size > 1 or force:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def all_reduce_mean(self, arrays, payload_bits=None):
        if len(arrays) != 1:
            raise ValueError(f"a distributed worker passes its own array only, got {len(arrays)}")
        t = arrays[0].detach().float().contiguous().clone()
        if self.world_size == 1:
            return t
        self.stats.bits_allreduced += 32 * t.numel() if payload_bits is None else payload_bits
        self.all_reduce_sum_(t)
        return t / self.world_size

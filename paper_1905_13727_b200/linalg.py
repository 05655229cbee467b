"""Errors and the Gram-Schmidt entry point of the reference's linalg layer.

`orthogonalize` is the drop-in for linalg.py:61-90 on the B200.  Float64 input
(numpy arrays, as the reference takes them, or float64 tensors) runs the
reference's modified Gram-Schmidt in float64 on the device with the seeded
replacement loop (`psgd_orthogonalize_f64`), so degenerate columns resolve
exactly as the reference resolves them; fp32 tensors run the hot path's K2
(`psgd_orthogonalize`: float64 arithmetic on fp32 input).  This wrapper only
moves data.
"""


class ContractViolation(ValueError):
    """An argument broke a documented precondition (linalg.py:20-21)."""


def orthogonalize(p, device=None):
    """linalg.py:61-90 on the GPU.  numpy in -> float64 numpy out; torch in -> torch
    out of the same dtype (float64 or float32)."""
    import numpy as np
    import torch

    from . import _lib
    from .plan import ptr, stream_ptr

    is_np = not isinstance(p, torch.Tensor)
    if is_np:
        a = np.asarray(p, dtype=np.float64)
        if a.ndim != 2:
            raise ContractViolation(f"orthogonalize input must be 2-d, got shape {a.shape}")
        if min(a.shape) < 1:
            raise ContractViolation(f"orthogonalize input has an empty dimension: {a.shape}")
        t = torch.from_numpy(np.ascontiguousarray(a)).to(device or "cuda")
    else:
        if p.dim() != 2 or min(p.shape) < 1:
            raise ContractViolation(f"orthogonalize input must be 2-d and non-empty, got {tuple(p.shape)}")
        dt = torch.float64 if p.dtype == torch.float64 else torch.float32
        t = p.detach().to(device=device or p.device, dtype=dt).contiguous().clone()
    n, r = t.shape
    if r > n:
        raise ContractViolation(f"cannot orthonormalize {r} columns in R^{n}")
    plan = _plan_for(n, r, t.device)
    status = torch.zeros(1, dtype=torch.int32, device=t.device)
    lib = _lib.lib()
    with torch.cuda.device(t.device):
        if t.dtype == torch.float64:
            out = torch.empty_like(t)
            _lib.check(lib.psgd_orthogonalize_f64(plan.handle, 0, ptr(t), ptr(plan.repl_table()), ptr(out),
                                                  ptr(status), stream_ptr()), "psgd_orthogonalize_f64")
        else:
            buf = torch.zeros(plan.p_elems, dtype=torch.float32, device=t.device)
            plan.p_view(buf, 0).copy_(t)
            _lib.check(lib.psgd_orthogonalize(plan.handle, ptr(buf), 1, ptr(plan.repl_table()),
                                              ptr(buf), None, ptr(status), stream_ptr()), "psgd_orthogonalize")
            out = plan.p_view(buf, 0).clone()
    st = int(status.item())
    if st & _lib.STATUS_NONFINITE_P:
        raise ContractViolation("orthogonalize input contains non-finite entries")
    if st & _lib.STATUS_REPLACEMENT:
        raise RuntimeError(f"Gram-Schmidt needed more than {_lib.REPL_ATTEMPTS} replacement draws for a column")
    return out.cpu().numpy() if is_np else out


_PLANS = {}


def _plan_for(n, r, device):
    from .plan import Plan
    key = (n, r, str(device))
    pl = _PLANS.get(key)
    if pl is None:
        pl = Plan([(n, r)], rank=r, world=1, nbias=0, device=device)
        _PLANS[key] = pl
    return pl

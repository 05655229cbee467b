"""Errors and the Gram-Schmidt entry point of the reference's linalg layer.

`orthogonalize` is the drop-in for linalg.py:61-90 on the B200: the float64
modified Gram-Schmidt with seeded degenerate-column replacement runs in the
K2 kernel (csrc/psgd_b200.cu:k2_gs); this wrapper only moves data.
"""


class ContractViolation(ValueError):
    """An argument broke a documented precondition (linalg.py:20-21)."""


def orthogonalize(p, device=None):
    """linalg.py:61-90 on the GPU.  numpy in -> float64 numpy out; torch in -> fp32 torch out."""
    import numpy as np
    import torch

    from . import _lib
    from .plan import Plan, ptr, stream_ptr

    is_np = not isinstance(p, torch.Tensor)
    if is_np:
        a = np.asarray(p, dtype=np.float64)
        if a.ndim != 2:
            raise ContractViolation(f"orthogonalize input must be 2-d, got shape {a.shape}")
        if min(a.shape) < 1:
            raise ContractViolation(f"orthogonalize input has an empty dimension: {a.shape}")
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(device or "cuda")
    else:
        if p.dim() != 2 or min(p.shape) < 1:
            raise ContractViolation(f"orthogonalize input must be 2-d and non-empty, got {tuple(p.shape)}")
        t = p.detach().to(device=device or p.device, dtype=torch.float32).contiguous().clone()
    n, r = t.shape
    if r > n:
        raise ContractViolation(f"cannot orthonormalize {r} columns in R^{n}")
    plan = _plan_for(n, r, t.device)
    buf = torch.zeros(plan.p_elems, dtype=torch.float32, device=t.device)
    plan.p_view(buf, 0).copy_(t)
    status = torch.zeros(1, dtype=torch.int32, device=t.device)
    with torch.cuda.device(t.device):
        _lib.check(_lib.lib().psgd_orthogonalize(plan.handle, ptr(buf), 1, ptr(plan.repl_table()),
                                                 ptr(buf), None, ptr(status), stream_ptr()), "psgd_orthogonalize")
    st = int(status.item())
    if st & _lib.STATUS_NONFINITE_P:
        raise ContractViolation("orthogonalize input contains non-finite entries")
    out = plan.p_view(buf, 0).clone()
    return out.double().cpu().numpy() if is_np else out


_PLANS = {}


def _plan_for(n, r, device):
    from .plan import Plan
    key = (n, r, str(device))
    pl = _PLANS.get(key)
    if pl is None:
        pl = Plan([(n, r)], rank=r, world=1, nbias=0, device=device)
        _PLANS[key] = pl
    return pl

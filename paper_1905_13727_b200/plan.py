"""Host-side mirror of the C plan: packed layout + per-plan device constants.

A plan fixes, for an ordered list of (n, m) matrices, the packed fp32 layout
of the flat gradient / error / work buffers (each matrix 16-B aligned), the
packed P (plus the uncompressed bias tail carried by the same all-reduce) and
Q buffers, and the kernels' work lists (see psgd_plan_create in
csrc/psgd_b200.cu).  It replaces the per-parameter Python loop of the
reference's optimizer.step (optimizer.py:110-129).
"""

import ctypes

import numpy as np
import torch

from . import _lib
from .seeding import replacement_column


class Plan:
    def __init__(self, shapes, rank, world=1, nbias=0, device=None):
        dev = torch.device(device if device is not None else "cuda")
        if dev.type == "cuda" and dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        if self.device.type != "cuda":
            raise ValueError(f"PowerSGD B200 plans live on a CUDA device, got {self.device}")
        lib = _lib.lib()
        shapes = [(int(n), int(m)) for n, m in shapes]
        nmat = len(shapes)
        ns = (ctypes.c_int64 * max(1, nmat))(*[s[0] for s in shapes])
        ms = (ctypes.c_int64 * max(1, nmat))(*[s[1] for s in shapes])
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(lib.psgd_plan_create(nmat, ns, ms, int(rank), int(world), int(nbias),
                                            ctypes.byref(handle)), "psgd_plan_create")
        self.handle = handle
        self._lib = lib
        info = _lib.PlanInfo()
        _lib.check(lib.psgd_plan_get_info(handle, ctypes.byref(info)), "psgd_plan_get_info")
        self.info = info
        self.shapes = shapes
        self.rank = int(rank)
        self.world = int(world)
        self.nbias = int(nbias)
        self.matrices = []
        for i in range(nmat):
            mi = _lib.MatrixInfo()
            _lib.check(lib.psgd_plan_matrix(handle, i, ctypes.byref(mi)), "psgd_plan_matrix")
            self.matrices.append(mi)
        self._repl = None

    # ------------------------------------------------------------------ sizes
    @property
    def flat_elems(self):
        return self.info.flat_elems

    @property
    def p_elems(self):
        return self.info.p_elems

    @property
    def q_elems(self):
        return self.info.q_elems

    @property
    def p_bias_off(self):
        return self.info.p_bias_off

    def repl_table(self):
        """linalg.py:54-58 replacement columns, float64 on the device: for every distinct
        row count n, column j of attempt a at repl_off + (a * repl_cols + j) * n
        (a < REPL_ATTEMPTS).  The draws depend on (n, j, attempt) only, so matrices
        with equal n share one table."""
        if self._repl is None:
            host = np.zeros(max(1, self.info.repl_elems), dtype=np.float64)
            done = set()
            for mi in self.matrices:
                if mi.repl_off in done:
                    continue
                done.add(mi.repl_off)
                for a in range(_lib.REPL_ATTEMPTS):
                    for j in range(mi.repl_cols):
                        o = mi.repl_off + (a * mi.repl_cols + j) * mi.n
                        host[o:o + mi.n] = replacement_column(mi.n, j, a)
            self._repl = torch.from_numpy(host).to(self.device)
        return self._repl

    # ------------------------------------------------------------------ views
    def matrix_view(self, flat, i):
        mi = self.matrices[i]
        return flat[mi.flat_off: mi.flat_off + mi.n * mi.m].view(mi.n, mi.m)

    def p_view(self, p, i):
        mi = self.matrices[i]
        return p[mi.p_off: mi.p_off + mi.n * mi.r_eff].view(mi.n, mi.r_eff)

    def q_view(self, q, i):
        """(m, r_eff) view of matrix i's Q; the packed block is column-major with
        column stride q_ld (so K1 reads it without smem bank conflicts)."""
        mi = self.matrices[i]
        return q[mi.q_off: mi.q_off + mi.r_eff * mi.q_ld].view(mi.r_eff, mi.q_ld)[:, :mi.m].t()

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            self._lib.psgd_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ptr(t):
    """Device pointer of a tensor (None -> NULL)."""
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)

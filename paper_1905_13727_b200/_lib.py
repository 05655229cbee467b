"""ctypes binding of `libpsgd_b200.so` (the C ABI declared in include/psgd_b200.h).

This module is the product's only route to compute: there is no CPU fallback.
If the library is missing or fails to load, importing it raises — loudly —
instead of degrading to another implementation.
"""

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpsgd_b200.so")

PSGD_OK = 0
PSGD_EINVAL = -1
PSGD_ECUDA = -2
PSGD_ENOMEM = -3

STATUS_NONFINITE_GRAD = 1
STATUS_NONFINITE_P = 2
STATUS_REPLACEMENT = 4

MAX_RANK = 16
MAX_TREE = 64
REPL_ATTEMPTS = 3  # PSGD_REPL_ATTEMPTS: replacement draws per column held on the device

# every symbol include/psgd_b200.h declares (tests check the export table)
EXPORTS = (
    "psgd_plan_create", "psgd_plan_destroy", "psgd_plan_get_info", "psgd_plan_matrix",
    "psgd_ef_p", "psgd_orthogonalize", "psgd_orthogonalize_f64", "psgd_q_ef", "psgd_decompress", "psgd_step_single",
    "psgd_tree_mean", "psgd_momentum_step", "psgd_step_single_sgd", "psgd_decompress_sgd",
    "psgd_last_error", "psgd_version",
)


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("flat_elems", ctypes.c_int64), ("p_elems", ctypes.c_int64),
        ("p_bias_off", ctypes.c_int64), ("q_elems", ctypes.c_int64),
        ("repl_elems", ctypes.c_int64), ("nbias", ctypes.c_int64),
        ("nmat", ctypes.c_int32), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
        ("n_tall", ctypes.c_int32), ("items_k1", ctypes.c_int64), ("items_k3", ctypes.c_int64),
        ("launches_ef_p", ctypes.c_int32), ("launches_orthogonalize", ctypes.c_int32),
        ("launches_q_ef", ctypes.c_int32), ("launches_decompress", ctypes.c_int32),
        ("launches_step_single", ctypes.c_int32), ("opt_fusable", ctypes.c_int32),
    ]


class Sgd(ctypes.Structure):
    """psgd_sgd: heavy-ball state of the fused update (optimizer.py:131-134)."""
    _fields_ = [
        ("params", ctypes.c_void_p), ("mom", ctypes.c_void_p), ("bias_params", ctypes.c_void_p),
        ("bias_mom", ctypes.c_void_p), ("lr", ctypes.c_float), ("momentum", ctypes.c_float),
        ("keep_update", ctypes.c_int32), ("pad", ctypes.c_int32),
    ]


class MatrixInfo(ctypes.Structure):
    _fields_ = [
        ("flat_off", ctypes.c_int64), ("p_off", ctypes.c_int64), ("q_off", ctypes.c_int64),
        ("repl_off", ctypes.c_int64), ("n", ctypes.c_int32), ("m", ctypes.c_int32),
        ("r_eff", ctypes.c_int32), ("tall", ctypes.c_int32), ("q_ld", ctypes.c_int32),
        ("repl_cols", ctypes.c_int32),
    ]


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64

_SIGNATURES = {
    "psgd_plan_create": (_I32, [_I32, ctypes.POINTER(_I64), ctypes.POINTER(_I64), _I32, _I32, _I64,
                                ctypes.POINTER(_P)]),
    "psgd_plan_destroy": (_I32, [_P]),
    "psgd_plan_get_info": (_I32, [_P, ctypes.POINTER(PlanInfo)]),
    "psgd_plan_matrix": (_I32, [_P, _I32, ctypes.POINTER(MatrixInfo)]),
    "psgd_ef_p": (_I32, [_P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "psgd_orthogonalize": (_I32, [_P, _P, _I32, _P, _P, _P, _P, _P]),
    "psgd_orthogonalize_f64": (_I32, [_P, _I32, _P, _P, _P, _P, _P]),
    "psgd_q_ef": (_I32, [_P, _P, _P, _I32, _P, _P, _P, _P, _P, _P, _P]),
    "psgd_decompress": (_I32, [_P, _P, _P, _I32, _P, _P, _P, _P]),
    "psgd_step_single": (_I32, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "psgd_tree_mean": (_I32, [ctypes.POINTER(_P), _I32, _I64, _P, _P]),
    "psgd_momentum_step": (_I32, [_P, _P, _P, _P, _P, _P, _P, ctypes.c_float, ctypes.c_float, _P, _P]),
    "psgd_step_single_sgd": (_I32, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, ctypes.c_void_p, _P, _P]),
    "psgd_decompress_sgd": (_I32, [_P, _P, _P, _I32, _P, _P, _P, ctypes.c_void_p, _P, _P]),
    "psgd_last_error": (ctypes.c_char_p, []),
    "psgd_version": (_I32, []),
}


def load(path=LIB_PATH):
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is deliberately no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = load(os.environ.get("PSGD_LIB", LIB_PATH))  # PSGD_LIB: an in-tree experiment build
    return _lib


class PsgdError(RuntimeError):
    """A CUDA-side failure reported by the library (PSGD_ECUDA / PSGD_ENOMEM)."""


def check(rc, what):
    if rc == PSGD_OK:
        return
    msg = lib().psgd_last_error().decode(errors="replace")
    if rc == PSGD_EINVAL:
        from .linalg import ContractViolation
        raise ContractViolation(f"{what}: {msg}")
    raise PsgdError(f"{what} failed ({rc}): {msg}")

"""Host-only check of the resident partition (no GPU): python tools/res_dryrun.py [workload] [rank]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_13727_b200 import _lib, catalogs  # noqa: E402


def dryrun(shapes, rank, nsm=148):
    n = (ctypes.c_int64 * len(shapes))(*[s[0] for s in shapes])
    m = (ctypes.c_int64 * len(shapes))(*[s[1] for s in shapes])
    st = (ctypes.c_double * 5)()
    why = ctypes.create_string_buffer(256)
    ok = _lib.lib().psgd_resident_dryrun(len(shapes), n, m, rank, nsm, st, why, 256)
    return ok, list(st), why.value.decode()


if __name__ == "__main__":
    wl = sys.argv[1] if len(sys.argv) > 1 else "resnet18"
    rank = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    shapes = [s.matrix_shape for s in catalogs.get_catalog(wl).params if not s.is_bias]
    print(dryrun(shapes, rank))

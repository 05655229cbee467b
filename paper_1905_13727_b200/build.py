"""Build the in-tree CUDA library `libpsgd_b200.so` for sm_100a with nvcc.

The .so lands next to this file so that it travels with the repo snapshot to
the GPU box (it is git-ignored, not gpurun-ignored)."""

import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SOURCES = [os.path.join(CSRC, "psgd_b200.cu")]
HEADERS = [os.path.join(CSRC, "common.cuh")]
LIB = os.path.join(HERE, "libpsgd_b200.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "--expt-relaxed-constexpr",
]


def nvcc_path():
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build libpsgd_b200.so")


def stale():
    if not os.path.exists(LIB):
        return True
    mt = os.path.getmtime(LIB)
    deps = SOURCES + HEADERS + [os.path.join(INCLUDE, "psgd_b200.h")]
    return any(os.path.getmtime(d) > mt for d in deps if os.path.exists(d))


def build(force=False, verbose=False, out=None, defines=()):
    """Compile csrc/*.cu -> libpsgd_b200.so (sm_100a).  Returns the path.
    `out` / `defines` build experiment variants (e.g. PSGD_PDL=0) beside it."""
    lib = out or LIB
    if not force and out is None and not stale():
        return LIB
    tmp = lib + ".tmp"
    nvcc = nvcc_path()
    objs, procs = [], []
    for src in SOURCES:  # translation units compile in parallel
        obj = f"{lib}.{os.path.basename(src)}.o"
        cmd = [nvcc, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", INCLUDE, "-c", "-o", obj, src]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        objs.append(obj)
        procs.append(subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    errs = []
    for p in procs:
        _, err = p.communicate()
        if p.returncode != 0:
            errs.append(f"nvcc failed ({p.returncode}):\n{err[-4000:]}")
        elif verbose:
            print(err)
    if errs:
        raise RuntimeError("\n".join(errs))
    res = subprocess.run([nvcc, "-shared", "-o", tmp, *objs, "-lcuda"], capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed ({res.returncode}):\n{res.stderr[-4000:]}")
    for o in objs:
        os.remove(o)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose=False))

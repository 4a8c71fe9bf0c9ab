"""Build the native library in-tree: paper_2010_13972_b200/_lib/libgts.so.

nvcc compiles the host C++ (path extraction, packers, blob writer) and the
sm_100a kernels into one shared library exporting the C ABI of include/gts.h.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIB_DIR, "libgts.so")
SOURCES = [os.path.join(CSRC, "host.cpp"), os.path.join(CSRC, "kernels.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("blob_format.h", "nodal.cuh", "warp_bins.cuh", "trace.h")] + [
    os.path.join(ROOT, "include", "gts.h")]

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xptxas", "-v",
    "-Xcompiler", "-fPIC,-fopenmp,-ffp-contract=off,-O3",
    "-shared",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Build libgts.so (or, with `out`/`defines`, a kernel variant for experiments)."""
    lib = os.path.abspath(out) if out else LIB
    if not force and out is None and not stale():
        return LIB
    os.makedirs(LIB_DIR, exist_ok=True)
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-o", tmp, *SOURCES, "-lgomp"]
    res = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    log = os.path.join(LIB_DIR, "build.log" if out is None else os.path.basename(lib) + ".log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))

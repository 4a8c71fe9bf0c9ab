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


# kernels.cu is compiled once per GTS_PART (0: the C ABI and small kernels;
# 1-4: the NODAL launches of {fp32, fp64} x {SHAP, interactions}) so that the
# heavy ptxas runs proceed in parallel; host.cpp is a sixth compile.
PARTS = (0, 1, 2, 3, 4)
COMPILE_FLAGS = [f for f in NVCC_FLAGS if f != "-shared"]


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Build libgts.so (or, with `out`/`defines`, a kernel variant for experiments)."""
    lib = os.path.abspath(out) if out else LIB
    if not force and out is None and not stale():
        return LIB
    os.makedirs(LIB_DIR, exist_ok=True)
    tag = f"{os.path.basename(lib)}.{os.getpid()}"
    objdir = os.path.join(LIB_DIR, "obj")
    os.makedirs(objdir, exist_ok=True)
    dflags = [f"-D{d}" for d in defines]
    jobs = []
    for part in PARTS:
        o = os.path.join(objdir, f"kernels{part}.{tag}.o")
        jobs.append((o, [nvcc(), *COMPILE_FLAGS, *dflags, f"-DGTS_PART={part}", "-c", "-o", o, SOURCES[1]]))
    o = os.path.join(objdir, f"host.{tag}.o")
    jobs.append((o, [nvcc(), *COMPILE_FLAGS, *dflags, "-c", "-o", o, SOURCES[0]]))
    procs = [(o, cmd, subprocess.Popen(cmd, cwd=CSRC, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
             for o, cmd in jobs]
    logs, ok = [], True
    for o, cmd, pr in procs:
        text, _ = pr.communicate()
        logs.append(" ".join(cmd) + "\n" + text)
        ok = ok and pr.returncode == 0
    tmp = lib + f".tmp{os.getpid()}"
    objs = [o for o, _ in jobs]
    if ok:
        # -z defs: an unresolved symbol (a missing part) fails the link instead of the first call
        cmd = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fopenmp",
               "-Xlinker", "-z,defs", "-o", tmp, *objs, "-lgomp"]
        res = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
        logs.append(" ".join(cmd) + "\n" + res.stdout + res.stderr)
        ok = res.returncode == 0
    for o in objs:
        if os.path.exists(o):
            os.remove(o)
    log = os.path.join(LIB_DIR, "build.log" if out is None else os.path.basename(lib) + ".log")
    with open(log, "w") as f:
        f.write("\n".join(logs))
    if not ok:
        sys.stderr.write("\n".join(logs)[-20000:])
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stderr.write("\n".join(logs))
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))

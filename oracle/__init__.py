"""oracle/ -- TEST INFRASTRUCTURE ONLY (not part of the product).

A plain, slow, obviously-correct CPU implementation of what the hot path
computes, written from the paper, sharing no code with
``paper_2010_13972_b200/``.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import it.

Contents (SURVEY.md §8(c) numbering):

* ``treeshap.c`` (O1, O5, O6): fp64 Algorithm 1 on the raw
  trees, conditioned recursion for interactions, predict,
  bias; OpenMP over rows (the paper's CPU baseline structure).
* ``brute.py`` (O2, O3, O4): cover-weighted f_S, Eq. 2 and
  Eq. 3/6 by subset enumeration.
* ``paths.py`` (O7, O8): independent path extraction + duplicate merge
   and bin packers, for byte-exact checks
  of the library's tables.
* ``closed_form.py`` (O9): per-path permutation-weight polynomial (derived from
  Eq. 2/3), a secondary check.

Parity status: every function here is pinned by tests/test_oracle_*.py (see
DESIGN.md "Oracle pins"); none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_oracle.so")
_SRC = os.path.join(_HERE, "treeshap.c")


def build(force: bool = False) -> str:
    """Compile treeshap.c (gcc, -O2, OpenMP) -> oracle/_oracle.so."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        model = [i64, vp, vp, vp, vp, vp, vp, vp, vp, i32, i32, dbl]
        for name in ("oracle_treeshap", "oracle_interactions", "oracle_predict"):
            fn = getattr(lib, name)
            fn.argtypes = model + [vp, i64, i64, vp]
            fn.restype = ctypes.c_int
        lib.oracle_bias.argtypes = model + [vp]
        lib.oracle_bias.restype = ctypes.c_int
        lib.oracle_extend_chain.argtypes = [ctypes.c_int, vp, vp, vp]
        lib.oracle_extend_chain.restype = ctypes.c_int
        lib.oracle_unwind_after_chain.argtypes = [ctypes.c_int, vp, vp, ctypes.c_int, vp]
        lib.oracle_unwind_after_chain.restype = ctypes.c_int
        lib.oracle_num_threads.argtypes = []
        lib.oracle_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _model_args(ens):
    keep = [np.ascontiguousarray(a) for a in (
        ens.node_offset.astype(np.int64), ens.left.astype(np.int32), ens.right.astype(np.int32),
        ens.feature.astype(np.int32), ens.threshold.astype(np.float32), ens.cover.astype(np.float64),
        ens.leaf_value.astype(np.float64), ens.tree_group.astype(np.int32))]
    args = [ens.n_trees] + [a.ctypes.data for a in keep] + [ens.n_features, ens.n_groups, float(ens.base_score)]
    return keep, args


def _x64(x):
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if x.ndim != 2:
        raise ValueError("X must be 2-D")
    return x


def treeshap(ens, x) -> np.ndarray:
    """O5: phi [n_rows][G][M+1] (bias at column M), fp64, Algorithm 1 on raw trees."""
    lib = _load()
    keep, args = _model_args(ens)
    x = _x64(x)
    out = np.empty((x.shape[0], ens.n_groups, ens.n_features + 1), np.float64)
    lib.oracle_treeshap(*args, x.ctypes.data, x.shape[0], x.shape[1], out.ctypes.data)
    return out


def interactions(ens, x) -> np.ndarray:
    """O6: phi_ij [n_rows][G][M+1][M+1], fp64, conditioned on/off recursion."""
    lib = _load()
    keep, args = _model_args(ens)
    x = _x64(x)
    M1 = ens.n_features + 1
    out = np.empty((x.shape[0], ens.n_groups, M1, M1), np.float64)
    lib.oracle_interactions(*args, x.ctypes.data, x.shape[0], x.shape[1], out.ctypes.data)
    return out


def predict(ens, x) -> np.ndarray:
    """O1: f(x) per group [n_rows][G]."""
    lib = _load()
    keep, args = _model_args(ens)
    x = _x64(x)
    out = np.empty((x.shape[0], ens.n_groups), np.float64)
    lib.oracle_predict(*args, x.ctypes.data, x.shape[0], x.shape[1], out.ctypes.data)
    return out


def bias(ens) -> np.ndarray:
    """E[f] per group (+ base_score), recursive cover weighting."""
    lib = _load()
    keep, args = _model_args(ens)
    out = np.empty(ens.n_groups, np.float64)
    lib.oracle_bias(*args, out.ctypes.data)
    return out


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def extend_chain(z, o) -> np.ndarray:
    """Weights after EXTENDing an empty list with (z[q], o[q]) for q = 0..n-1
    (PAPER.md:79-88); element 0 is the root seed."""
    z = np.ascontiguousarray(z, np.float64); o = np.ascontiguousarray(o, np.float64)
    out = np.empty(len(z), np.float64)
    if _load().oracle_extend_chain(len(z), z.ctypes.data, o.ctypes.data, out.ctypes.data) != 0:
        raise ValueError("bad chain")
    return out


def unwind_after_chain(z, o, i) -> np.ndarray:
    """Weights after UNWINDing 1-based element i from extend_chain(z, o)."""
    z = np.ascontiguousarray(z, np.float64); o = np.ascontiguousarray(o, np.float64)
    out = np.empty(max(len(z) - 1, 0), np.float64)
    if _load().oracle_unwind_after_chain(len(z), z.ctypes.data, o.ctypes.data, int(i), out.ctypes.data) != 0:
        raise ValueError("bad unwind")
    return out

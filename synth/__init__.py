"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module holds NONE of the method's arithmetic (no path extraction, no
Shapley weights, no packing).  It only produces the inputs the method consumes:

* ``Ensemble``: a tree ensemble as the node lists {v, a, b, t, r, d} of
  PAPER.md:114 (Algorithm 1 context), flattened CSR-over-trees exactly as the
  C ABI takes them (include/gts.h, ``gts_model``);
* ``make_ensemble``: random-split ensembles grown by ``_synth.c`` (recipe in its
  header and in DESIGN.md "Input recipe");
* ``make_x``: counter-keyed U[0,1) fp32 feature matrices, any row shard
  reproducible on its own;
* small hand-built fixtures from SPEC.md (stump, depth-2) used by the pins.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_synth.so")
_SRC = os.path.join(_HERE, "_synth.c")


def build(force: bool = False) -> str:
    """Compile _synth.c with gcc (OpenMP) into synth/_synth.so."""
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
        i64, i32, dbl, u64, vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_uint64, ctypes.c_void_p
        lib.synth_grow_ensemble.argtypes = [i64, i32, i32, i32, dbl, dbl, dbl, dbl, u64, dbl, i64,
                                            vp, vp, vp, vp, vp, vp, vp]
        lib.synth_grow_ensemble.restype = ctypes.c_int
        lib.synth_fill_x_f32.argtypes = [u64, i64, i64, i32, vp]
        lib.synth_fill_x_f32.restype = None
        _lib = lib
    return _lib


@dataclass
class Ensemble:
    """Tree ensemble as flat node lists (v=leaf_value, a=left,
    b=right, t=threshold, r=cover, d=feature).  Local node 0 of each tree is its
    root; children are local indices, -1 at leaves.  Split rule: x < t -> left."""

    node_offset: np.ndarray  # int64 [T+1]
    left: np.ndarray  # int32 [N]
    right: np.ndarray  # int32 [N]
    feature: np.ndarray  # int32 [N] (-1 at leaves)
    threshold: np.ndarray  # float32 [N]
    cover: np.ndarray  # float64 [N]
    leaf_value: np.ndarray  # float64 [N]
    tree_group: np.ndarray  # int32 [T]
    n_features: int
    n_groups: int
    base_score: float = 0.0
    meta: dict = field(default_factory=dict)

    @property
    def n_trees(self) -> int:
        return int(self.node_offset.shape[0] - 1)

    @property
    def n_nodes(self) -> int:
        return int(self.node_offset[-1])

    def tree(self, t: int):
        """Local arrays of tree t: (left, right, feature, threshold, cover, leaf_value)."""
        a, b = int(self.node_offset[t]), int(self.node_offset[t + 1])
        return (self.left[a:b], self.right[a:b], self.feature[a:b], self.threshold[a:b],
                self.cover[a:b], self.leaf_value[a:b])

    def n_leaves(self) -> int:
        return int(np.count_nonzero(self.left < 0))

    def subset(self, trees) -> "Ensemble":
        """A new ensemble made of the listed trees (in the given order)."""
        trees = [int(t) for t in trees]
        parts = [(int(self.node_offset[t]), int(self.node_offset[t + 1])) for t in trees]
        idx = np.concatenate([np.arange(a, b) for a, b in parts]) if parts else np.zeros(0, np.int64)
        sizes = np.array([b - a for a, b in parts], dtype=np.int64)
        off = np.zeros(len(trees) + 1, dtype=np.int64)
        off[1:] = np.cumsum(sizes)
        return Ensemble(off, self.left[idx].copy(), self.right[idx].copy(), self.feature[idx].copy(),
                        self.threshold[idx].copy(), self.cover[idx].copy(), self.leaf_value[idx].copy(),
                        self.tree_group[trees].copy(), self.n_features, self.n_groups, self.base_score,
                        dict(self.meta))


def ensemble_from_trees(trees, n_features: int, n_groups: int = 1, groups=None,
                        base_score: float = 0.0) -> Ensemble:
    """Build an Ensemble from per-tree node dicts.

    Each tree is a list of nodes; node i is a dict with either
    ``{"feature", "threshold", "left", "right", "cover"}`` (internal) or
    ``{"leaf_value", "cover"}`` (leaf).  Node 0 is the root.
    """
    L, R, F, TH, C, V = [], [], [], [], [], []
    off = [0]
    for nodes in trees:
        for nd in nodes:
            if "leaf_value" in nd:
                L.append(-1); R.append(-1); F.append(-1); TH.append(0.0)
                V.append(float(nd["leaf_value"]))
            else:
                L.append(int(nd["left"])); R.append(int(nd["right"])); F.append(int(nd["feature"]))
                TH.append(float(nd["threshold"])); V.append(0.0)
            C.append(float(nd["cover"]))
        off.append(off[-1] + len(nodes))
    if groups is None:
        groups = [t % n_groups for t in range(len(trees))]
    return Ensemble(np.array(off, np.int64), np.array(L, np.int32), np.array(R, np.int32),
                    np.array(F, np.int32), np.array(TH, np.float32), np.array(C, np.float64),
                    np.array(V, np.float64), np.array(groups, np.int32), n_features, n_groups,
                    float(base_score))


def make_ensemble(n_trees: int, n_features: int, max_depth: int, leaves_per_tree: float,
                  n_groups: int = 1, zipf_s: float = 1.0, beta: float = 0.0, seed: int = 0,
                  root_cover: float = float(1 << 20), base_score: float = 0.0,
                  cover_skew: float = 0.0) -> Ensemble:
    """Random-split ensemble (recipe: synth/_synth.c header).  Tree t belongs to
    group t mod n_groups (XGBoost round-robin).  cover_skew > 0
    draws skewed cover splits (zero fractions down to cover_skew); pair it with
    a large root_cover (e.g. 2**50) so deep nodes keep integer covers >= 2."""
    lib = _load()
    lf = int(np.floor(leaves_per_tree))
    frac = float(leaves_per_tree - lf)
    max_leaves = min(lf + 1, 1 << max_depth)
    max_nodes = 2 * max_leaves - 1
    T = int(n_trees)
    shape = (T * max_nodes,)
    left = np.empty(shape, np.int32); right = np.empty(shape, np.int32)
    feat = np.empty(shape, np.int32); thr = np.empty(shape, np.float32)
    cov = np.empty(shape, np.float64); val = np.empty(shape, np.float64)
    nn = np.zeros(T, np.int64)
    rc = lib.synth_grow_ensemble(T, n_features, max_depth, lf, frac, zipf_s, beta, root_cover,
                                 ctypes.c_uint64(seed & (2**64 - 1)), float(cover_skew), max_nodes,
                                 left.ctypes.data, right.ctypes.data, feat.ctypes.data, thr.ctypes.data,
                                 cov.ctypes.data, val.ctypes.data, nn.ctypes.data)
    if rc != 0:
        raise RuntimeError("synth_grow_ensemble failed")
    keep = (np.arange(max_nodes)[None, :] < nn[:, None]).reshape(-1)
    off = np.zeros(T + 1, np.int64)
    off[1:] = np.cumsum(nn)
    groups = (np.arange(T) % n_groups).astype(np.int32)
    return Ensemble(off, left[keep], right[keep], feat[keep], thr[keep], cov[keep], val[keep], groups,
                    int(n_features), int(n_groups), float(base_score),
                    dict(n_trees=T, max_depth=max_depth, leaves_per_tree=leaves_per_tree,
                         zipf_s=zipf_s, beta=beta, seed=seed, cover_skew=cover_skew))


def make_x(seed: int, n_rows: int, n_features: int, row0: int = 0) -> np.ndarray:
    """Rows [row0, row0+n_rows) of the counter-keyed U[0,1) fp32 matrix."""
    lib = _load()
    out = np.empty((int(n_rows), int(n_features)), np.float32)
    if n_rows > 0:
        lib.synth_fill_x_f32(ctypes.c_uint64(seed & (2**64 - 1)), int(row0), int(n_rows),
                             int(n_features), out.ctypes.data)
    return out


def inject_ties(x: np.ndarray, ens: Ensemble, frac: float, seed: int) -> np.ndarray:
    """Set about ``frac`` of the entries exactly equal to a split threshold used on
    that feature (the x == t tie case of reading G1, PAPER.md:68 vs 197)."""
    rng = np.random.default_rng(seed)
    x = x.copy()
    internal = ens.left >= 0
    by_f = {}
    for f, t in zip(ens.feature[internal], ens.threshold[internal]):
        by_f.setdefault(int(f), []).append(np.float32(t))
    mask = rng.random(x.shape) < frac
    for r, c in zip(*np.nonzero(mask)):
        ts = by_f.get(int(c))
        if ts:
            x[r, c] = ts[int(rng.integers(len(ts)))]
    return x


# ----------------------------------------------------------------------------
# hand-built fixtures (SPEC.md worked examples)
# ----------------------------------------------------------------------------

def stump() -> Ensemble:
    """root f0 < 0.5 cover 10, leaves v=1.0 cover 4 / v=0.0 cover 6."""
    return ensemble_from_trees([[
        {"feature": 0, "threshold": 0.5, "left": 1, "right": 2, "cover": 10.0},
        {"leaf_value": 1.0, "cover": 4.0},
        {"leaf_value": 0.0, "cover": 6.0},
    ]], n_features=1)


def depth2() -> Ensemble:
    """root f0<0.5 cover 10; left child f1<0.5 cover 4 with leaves
    v=1 cover 1, v=2 cover 3; right leaf v=0 cover 6."""
    return ensemble_from_trees([[
        {"feature": 0, "threshold": 0.5, "left": 1, "right": 2, "cover": 10.0},
        {"feature": 1, "threshold": 0.5, "left": 3, "right": 4, "cover": 4.0},
        {"leaf_value": 0.0, "cover": 6.0},
        {"leaf_value": 1.0, "cover": 1.0},
        {"leaf_value": 2.0, "cover": 3.0},
    ]], n_features=2)


def single_leaf(v: float = 0.7) -> Ensemble:
    """a tree that is one leaf."""
    return ensemble_from_trees([[{"leaf_value": v, "cover": 10.0}]], n_features=1)

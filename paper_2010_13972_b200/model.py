"""Tree-ensemble input for the C ABI, and ingestion of XGBoost `dump_model`
JSON.

`TreeModel` holds the paper's per-node lists {v, a, b, t, r, d}
in the CSR-over-trees layout that `gts_model` (include/gts.h) takes: tree t
owns nodes [node_offset[t], node_offset[t+1]), local node 0 is its root,
children are local indices (-1 at leaves), split rule x < t -> left.  The
library validates the model (gts_extract_paths); this module only parses.
"""
from __future__ import annotations

import json
import re
from dataclasses import dataclass

import numpy as np


@dataclass
class TreeModel:
    node_offset: np.ndarray  # int64 [T+1]
    left: np.ndarray  # int32 [N]  a_j
    right: np.ndarray  # int32 [N]  b_j
    feature: np.ndarray  # int32 [N]  d_j (-1 at leaves)
    threshold: np.ndarray  # float32 [N]  t_j
    cover: np.ndarray  # float64 [N]  r_j
    leaf_value: np.ndarray  # float64 [N]  v_j
    tree_group: np.ndarray  # int32 [T]
    n_features: int
    n_groups: int
    base_score: float = 0.0
    cover_adjust: float = 0.0  # largest relative change made by covers="conserve" (0 = none)

    @property
    def n_trees(self) -> int:
        return int(self.node_offset.shape[0] - 1)

    def tree(self, t: int):
        """Local arrays of tree t: (left, right, feature, threshold, cover, leaf_value)."""
        a, b = int(self.node_offset[t]), int(self.node_offset[t + 1])
        return (self.left[a:b], self.right[a:b], self.feature[a:b], self.threshold[a:b],
                self.cover[a:b], self.leaf_value[a:b])


class DumpError(ValueError):
    """A dump that violates the format's preconditions."""


_FNAME = re.compile(r"^f(\d+)$")


def _feature_index(name, feature_map, where):
    if isinstance(name, int):
        return name
    if feature_map is not None:
        if name not in feature_map:
            raise DumpError(f"{where}: split feature {name!r} is not in the feature map")
        return int(feature_map[name])
    m = _FNAME.match(str(name))
    if not m:
        raise DumpError(f"{where}: split name {name!r} is not of the form f<k> and no feature map was given")
    return int(m.group(1))


def _conserve_covers(left, right, cover):
    """Internal covers := sum of their children's, bottom-up in fp64 (root
    first ordering: every child index is larger than its parent's).  Returns
    the largest relative change."""
    worst = 0.0
    for j in range(len(left) - 1, -1, -1):
        if left[j] >= 0:
            c = cover[left[j]] + cover[right[j]]
            worst = max(worst, abs(c - cover[j]) / c)
            cover[j] = c
    return worst


def from_xgboost_dump(doc, num_class: int = 1, feature_map=None, n_features: int | None = None,
                      base_score: float = 0.0, covers: str = "conserve", cover_rtol: float = 1e-4) -> TreeModel:
    """Parse XGBoost `Booster.dump_model(..., dump_format="json")` output.

    doc: the JSON text, or the already-parsed list of tree objects.  Each node
    is {"nodeid", "split", "split_condition", "yes", "no", "missing", "cover",
    "children"} or a leaf {"nodeid", "leaf", "cover"}; x < split_condition takes
    "yes".  Tree i belongs to group i mod num_class (round robin,
    SPEC.md:63).  feature_map maps split names to indices when they are not
    "f<k>".  n_features defaults to 1 + the largest split index.  A "missing"
    branch that is neither "yes" nor "no" is rejected (X must be finite, G17).

    covers: XGBoost stores each node's hessian sum as float32 and the dump
    prints it at limited precision, so a parent's printed cover differs from
    the sum of its children's by up to ~1e-6 relative -- at or beyond the
    library's 1e-6 conservation check.  "conserve" (default)
    rebuilds every internal cover as the sum of its children's, bottom-up in
    fp64 from the printed leaf covers (the relative change, ~1e-7, is kept in
    ``cover_adjust``; z = r_child / r_parent then changes by as much, far below
    fp32 kernel rounding); "as_is" passes the printed covers through, and the
    library rejects the model if they do not conserve.  A printed cover that
    is off by more than cover_rtol (relative) is a broken dump, not rounding:
    DumpError.
    """
    if covers not in ("conserve", "as_is"):
        raise DumpError("covers must be 'conserve' or 'as_is'")
    trees = json.loads(doc) if isinstance(doc, (str, bytes)) else doc
    if not isinstance(trees, list):
        raise DumpError("dump must be a JSON array of tree objects")
    if num_class < 1:
        raise DumpError("num_class must be >= 1")
    L, R, F, TH, C, V, off = [], [], [], [], [], [], [0]
    max_f = -1
    adjust = 0.0
    for t, root in enumerate(trees):
        nodes = {}
        stack = [root]
        while stack:  # collect every node object of the tree by id
            nd = stack.pop()
            if not isinstance(nd, dict) or "nodeid" not in nd:
                raise DumpError(f"tree {t}: node without nodeid")
            nid = int(nd["nodeid"])
            if nid in nodes:
                raise DumpError(f"tree {t}: duplicate nodeid {nid}")
            nodes[nid] = nd
            stack.extend(nd.get("children", []))
        # local order: root first, then depth-first (yes before no)
        order, local = [], {}
        stack = [int(root["nodeid"])]
        while stack:
            nid = stack.pop()
            if nid not in nodes:
                raise DumpError(f"tree {t}: dangling child id {nid}")
            if nid in local:
                raise DumpError(f"tree {t}: node {nid} reached twice")
            local[nid] = len(order)
            order.append(nid)
            nd = nodes[nid]
            if "leaf" not in nd:
                stack.append(int(nd["no"]))
                stack.append(int(nd["yes"]))
        c0 = len(C)
        for nid in order:
            nd = nodes[nid]
            where = f"tree {t} node {nid}"
            if "cover" not in nd:
                raise DumpError(f"{where}: missing cover")
            C.append(float(nd["cover"]))
            if "leaf" in nd:
                L.append(-1); R.append(-1); F.append(-1); TH.append(0.0); V.append(float(nd["leaf"]))
                continue
            for k in ("split", "split_condition", "yes", "no"):
                if k not in nd:
                    raise DumpError(f"{where}: missing {k}")
            yes, no = int(nd["yes"]), int(nd["no"])
            if "missing" in nd and int(nd["missing"]) not in (yes, no):
                raise DumpError(f"{where}: missing-branch id {nd['missing']} is neither yes nor no")
            f = _feature_index(nd["split"], feature_map, where)
            max_f = max(max_f, f)
            L.append(local[yes]); R.append(local[no]); F.append(f)
            TH.append(float(nd["split_condition"])); V.append(0.0)
        if covers == "conserve":
            lt, rt, ct = L[c0:], R[c0:], C[c0:]
            worst = _conserve_covers(lt, rt, ct)
            if worst > cover_rtol:
                raise DumpError(f"tree {t}: cover(parent) differs from cover(left) + cover(right) by "
                                f"{worst:.3g} relative (> cover_rtol {cover_rtol:g})")
            adjust = max(adjust, worst)
            C[c0:] = ct
        off.append(off[-1] + len(order))
    m = (max_f + 1) if n_features is None else int(n_features)
    return TreeModel(np.array(off, np.int64), np.array(L, np.int32), np.array(R, np.int32),
                     np.array(F, np.int32), np.array(TH, np.float32), np.array(C, np.float64),
                     np.array(V, np.float64), np.array([t % num_class for t in range(len(trees))], np.int32),
                     max(m, 1), int(num_class), float(base_score), float(adjust))

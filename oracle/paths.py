"""oracle/paths.py -- TEST INFRASTRUCTURE ONLY.

Independent re-statement of the preprocessing steps,
for byte-exact checks of the library's tables.  Plain Python loops.

O7  extract_paths (§3.1; Listing 1) and the
    duplicate merge (§3.2):
    * trees in input order; within a tree, leaves in DFS left-first order (G9);
    * a path = root element (feature -1, [-inf, +inf), z = 1) then one element
      per edge parent->child: the parent's feature, [-inf, t) for the left
      child or [t, +inf) for the right child (x < t -> left, G1), and
      z = cover(child) / cover(parent) in fp64;
    * merge: stable sort of the non-root elements by feature (root first, G10);
      a run of equal features becomes one element with lower = max, upper =
      min, z = product of the run's z in root-to-leaf order, fp64 (G11);
    * bias_g = sum over the group's paths, in path order, of v * prod(z over the
      path's elements in table order), fp64, then + base_score (G13).
O8  packers (§3.3; utilisation PAPER.md:455):
    items are paths, size = merged length (root lane included), capacity B;
    FFD / BFD order = stable sort by size descending, ties by path index;
    bins are numbered by creation; FFD takes the lowest-index bin with residual
    >= size, BFD the bin with the smallest residual >= size (ties: lowest index)
    (G12).  Implemented with 33 per-residual min-heaps of bin ids -- deliberately
    a different data structure from the library's.  NF keeps one open bin in
    arrival (path) order; "none" gives every path its own bin.  A path occupies
    consecutive lanes of its bin in insertion order from lane 0.
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass

import numpy as np

NEG_INF = np.float32(-np.inf)
POS_INF = np.float32(np.inf)


@dataclass
class PathTable:
    path_offset: np.ndarray  # int64 [L+1]
    feature: np.ndarray  # int32 [E]
    lower: np.ndarray  # float32 [E]
    upper: np.ndarray  # float32 [E]
    zero_fraction: np.ndarray  # float64 [E]
    v: np.ndarray  # float64 [L]
    group: np.ndarray  # int32 [L]
    tree: np.ndarray  # int32 [L]
    bias: np.ndarray  # float64 [G]

    @property
    def n_paths(self):
        return int(self.path_offset.shape[0] - 1)

    def lengths(self):
        return np.diff(self.path_offset).astype(np.int64)


def _tree_paths(left, right, feat, thr, cov, val):
    """Raw (unmerged) paths of one tree, DFS left-first.  Yields (elements, v);
    each element = (feature, lower, upper, z)."""
    out = []
    # explicit stack of (node, edges-so-far); push right then left so left pops first
    stack = [(0, [])]
    while stack:
        j, edges = stack.pop()
        if left[j] < 0:
            out.append((edges, float(val[j])))
            continue
        a, b, f, t = int(left[j]), int(right[j]), int(feat[j]), np.float32(thr[j])
        rj = float(cov[j])
        right_edge = (f, t, POS_INF, float(cov[b]) / rj)
        left_edge = (f, NEG_INF, t, float(cov[a]) / rj)
        stack.append((b, edges + [right_edge]))
        stack.append((a, edges + [left_edge]))
    return out


def merge(edges):
    """Duplicate merge of one path's non-root edges (stable sort by feature)."""
    order = sorted(range(len(edges)), key=lambda q: edges[q][0])  # Python sort is stable
    merged = []
    for q in order:
        f, lo, hi, z = edges[q]
        if merged and merged[-1][0] == f:
            pf, plo, phi, pz = merged[-1]
            merged[-1] = (f, max(plo, lo), min(phi, hi), pz * z)
        else:
            merged.append((f, lo, hi, z))
    return merged


def extract_paths(ens) -> PathTable:
    offs = [0]
    F, LO, HI, Z, V, G, T = [], [], [], [], [], [], []
    for t in range(ens.n_trees):
        left, right, feat, thr, cov, val = ens.tree(t)
        for edges, v in _tree_paths(left, right, feat, thr, cov, val):
            els = [(-1, NEG_INF, POS_INF, 1.0)] + merge(edges)
            for f, lo, hi, z in els:
                F.append(f); LO.append(lo); HI.append(hi); Z.append(z)
            offs.append(offs[-1] + len(els))
            V.append(v); G.append(int(ens.tree_group[t])); T.append(t)
    tab = PathTable(np.array(offs, np.int64), np.array(F, np.int32), np.array(LO, np.float32),
                    np.array(HI, np.float32), np.array(Z, np.float64), np.array(V, np.float64),
                    np.array(G, np.int32), np.array(T, np.int32), np.zeros(ens.n_groups, np.float64))
    tab.bias = path_bias(tab, ens.n_groups, ens.base_score)
    return tab


def path_bias(tab: PathTable, n_groups: int, base_score: float) -> np.ndarray:
    """bias_g = sum_paths v * prod z (path order, table order), + base_score last."""
    acc = [0.0] * n_groups
    z = tab.zero_fraction.tolist()
    off = tab.path_offset.tolist()
    for p in range(tab.n_paths):
        prod = 1.0
        for e in range(off[p], off[p + 1]):
            prod *= z[e]
        acc[int(tab.group[p])] += float(tab.v[p]) * prod
    return np.array([a + float(base_score) for a in acc], np.float64)


# ----------------------------------------------------------------------------
# packers
# ----------------------------------------------------------------------------

@dataclass
class Packing:
    bin_of_item: np.ndarray  # int32 [n]
    lane_of_item: np.ndarray  # uint8 [n]
    n_bins: int
    sum_sizes: int
    capacity: int

    @property
    def utilisation(self):
        return 1.0 if self.n_bins == 0 else self.sum_sizes / (self.capacity * self.n_bins)


def _finish(sizes, bins_in_order, n_bins, capacity):
    n = len(sizes)
    bin_of = np.zeros(n, np.int32)
    lane_of = np.zeros(n, np.uint8)
    fill = [0] * n_bins
    for i, b in bins_in_order:
        bin_of[i] = b
        lane_of[i] = fill[b]
        fill[b] += int(sizes[i])
    return Packing(bin_of, lane_of, n_bins, int(np.sum(sizes, dtype=np.int64)), capacity)


def _check(sizes, capacity):
    for s in sizes:
        if s < 1 or s > capacity:
            raise ValueError(f"item size {s} outside [1, {capacity}]")


def decreasing_order(sizes):
    return sorted(range(len(sizes)), key=lambda i: (-int(sizes[i]), i))


def pack_ffd(sizes, capacity=32) -> Packing:
    return _pack_fit(sizes, capacity, best=False)


def pack_bfd(sizes, capacity=32) -> Packing:
    return _pack_fit(sizes, capacity, best=True)


def _pack_fit(sizes, capacity, best):
    _check(sizes, capacity)
    heaps = [[] for _ in range(capacity + 1)]  # heaps[r] = min-heap of bin ids with residual r
    n_bins = 0
    placed = []
    for i in decreasing_order(sizes):
        s = int(sizes[i])
        choice_r = -1
        if best:
            for r in range(s, capacity + 1):
                if heaps[r]:
                    choice_r = r
                    break
        else:
            best_id = None
            for r in range(s, capacity + 1):
                if heaps[r] and (best_id is None or heaps[r][0] < best_id):
                    best_id, choice_r = heaps[r][0], r
        if choice_r < 0:
            b = n_bins
            n_bins += 1
            r_new = capacity - s
        else:
            b = heapq.heappop(heaps[choice_r])
            r_new = choice_r - s
        heapq.heappush(heaps[r_new], b)
        placed.append((i, b))
    return _finish(sizes, placed, n_bins, capacity)


def pack_nf(sizes, capacity=32) -> Packing:
    _check(sizes, capacity)
    placed = []
    n_bins = 0
    fill = capacity + 1
    for i, s in enumerate(sizes):
        s = int(s)
        if fill + s > capacity:
            n_bins += 1
            fill = 0
        placed.append((i, n_bins - 1))
        fill += s
    return _finish(sizes, placed, n_bins, capacity)


def pack_none(sizes, capacity=32) -> Packing:
    _check(sizes, capacity)
    return _finish(sizes, [(i, i) for i in range(len(sizes))], len(sizes), capacity)


def opt_bins(sizes, capacity=32, max_items=32) -> int:
    """Minimal number of bins by exhaustive search (small n)."""
    sizes = sorted((int(s) for s in sizes), reverse=True)
    if len(sizes) > max_items:
        raise ValueError("instance too large for brute force")
    _check(sizes, capacity)
    best = [len(sizes)]

    def rec(i, loads):
        if len(loads) >= best[0]:
            return
        if i == len(sizes):
            best[0] = len(loads)
            return
        s = sizes[i]
        seen = set()
        for b in range(len(loads)):
            if loads[b] + s <= capacity and loads[b] not in seen:
                seen.add(loads[b])
                loads[b] += s
                rec(i + 1, loads)
                loads[b] -= s
        loads.append(s)
        rec(i + 1, loads)
        loads.pop()

    rec(0, [])
    return best[0]

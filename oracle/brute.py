"""oracle/brute.py -- TEST INFRASTRUCTURE ONLY.

Definitions written out, by subset enumeration (pure Python, fp64, small M):

* ``cond_expect`` (O2): f_S(x) = E[f(x) | x_S] with cover weighting
  (PAPER.md:50): at a split on a feature in S follow x (x < t -> left,
  reading G1); otherwise average both children weighted by their covers.
* ``shap_values`` (O3): Eq. 2 over the features U split on by
  the group's trees (features outside U are dummies with phi = 0, SPEC.md:330,
  reading G22); bias phi_0 = f_empty + base_score (Eq. 1).
* ``interaction_values`` (O4): Eq. 3 for i != j, Eq. 6
   for the diagonal; cell (M,M) = bias, (i,M) = (M,i) = 0
  (reading G14).
"""
from __future__ import annotations

from itertools import combinations
from math import factorial

import numpy as np


def _tree_lists(ens, t):
    a, b = int(ens.node_offset[t]), int(ens.node_offset[t + 1])
    return (ens.left[a:b].tolist(), ens.right[a:b].tolist(), ens.feature[a:b].tolist(),
            [float(v) for v in ens.threshold[a:b]], ens.cover[a:b].tolist(), ens.leaf_value[a:b].tolist())


def _expect_tree(tl, x, S, j=0):
    left, right, feat, thr, cov, val = tl
    if left[j] < 0:
        return val[j]
    a, b = left[j], right[j]
    if feat[j] in S:
        return _expect_tree(tl, x, S, a if x[feat[j]] < thr[j] else b)
    return (cov[a] * _expect_tree(tl, x, S, a) + cov[b] * _expect_tree(tl, x, S, b)) / cov[j]


def cond_expect(ens, x, S, group=0):
    """f_S(x) for one group: base_score + sum over the group's trees (O2)."""
    S = frozenset(S)
    total = float(ens.base_score)
    for t in range(ens.n_trees):
        if int(ens.tree_group[t]) == group:
            total += _expect_tree(_tree_lists(ens, t), x, S)
    return total


def used_features(ens, group=0):
    U = set()
    for t in range(ens.n_trees):
        if int(ens.tree_group[t]) == group:
            a, b = int(ens.node_offset[t]), int(ens.node_offset[t + 1])
            for q in range(a, b):
                if ens.left[q] >= 0:
                    U.add(int(ens.feature[q]))
    return sorted(U)


def _all_f(ens, x, U, group):
    """f_S for every subset S of U, keyed by frozenset."""
    x = [float(v) for v in x]
    tls = [_tree_lists(ens, t) for t in range(ens.n_trees) if int(ens.tree_group[t]) == group]
    table = {}
    for r in range(len(U) + 1):
        for S in combinations(U, r):
            fs = frozenset(S)
            table[fs] = float(ens.base_score) + sum(_expect_tree(tl, x, fs) for tl in tls)
    return table


def shap_values(ens, x, group=0, max_features=12):
    """Eq. 2 for one row and group: array [M+1], bias at index M."""
    U = used_features(ens, group)
    if len(U) > max_features:
        raise ValueError(f"brute force limited to {max_features} used features, got {len(U)}")
    f = _all_f(ens, x, U, group)
    M = ens.n_features
    n = len(U)
    phi = np.zeros(M + 1)
    for i in U:
        rest = [u for u in U if u != i]
        s = 0.0
        for r in range(len(rest) + 1):
            w = factorial(r) * factorial(n - r - 1) / factorial(n)
            for S in combinations(rest, r):
                fs = frozenset(S)
                s += w * (f[fs | {i}] - f[fs])
        phi[i] = s
    phi[M] = f[frozenset()]
    return phi


def interaction_values(ens, x, group=0, max_features=10):
    """Eq. 3 / Eq. 6 for one row and group: matrix [M+1][M+1]."""
    U = used_features(ens, group)
    if len(U) > max_features:
        raise ValueError(f"brute force limited to {max_features} used features, got {len(U)}")
    f = _all_f(ens, x, U, group)
    M = ens.n_features
    n = len(U)
    mat = np.zeros((M + 1, M + 1))
    for i in U:
        for j in U:
            if i == j:
                continue
            rest = [u for u in U if u != i and u != j]
            s = 0.0
            for r in range(len(rest) + 1):
                w = factorial(r) * factorial(n - r - 2) / (2.0 * factorial(n - 1))
                for S in combinations(rest, r):
                    fs = frozenset(S)
                    s += w * (f[fs | {i, j}] - f[fs | {i}] - f[fs | {j}] + f[fs])
            mat[i, j] = s
    phi = shap_values(ens, x, group, max_features)
    for i in U:
        mat[i, i] = phi[i] - sum(mat[i, j] for j in U if j != i)
    mat[M, M] = f[frozenset()]
    return mat

"""oracle/closed_form.py -- TEST INFRASTRUCTURE ONLY.

O9: the per-path closed form behind
EXTEND/UNWIND, derived from Eq. 2/3 and leaf
additivity.  For a merged path with non-root elements F
(|F| = k), leaf value v, zero fractions z_s and one fractions
o_s = [lower_s <= x_{d_s} < upper_s]:

  phi_i  = v (o_i - z_i) * sum_{m=0}^{k-1} m!(k-1-m)!/k! * [t^m] prod_{s in F\\i}(z_s + o_s t)
  phi_ij = 1/2 v (o_i - z_i)(o_j - z_j)
           * sum_{m=0}^{k-2} m!(k-2-m)!/(k-1)! * [t^m] prod_{s in F\\{i,j}}(z_s + o_s t)

The polynomial coefficients are built by explicit convolution (fp64).  Works on
an ``oracle.paths.PathTable``; output layouts as the kernels' (bias at column M).
"""
from __future__ import annotations

from math import factorial

import numpy as np


def _poly(zs, os_):
    c = np.array([1.0])
    for z, o in zip(zs, os_):
        c = np.convolve(c, np.array([z, o]))
    return c


def _weights(n):
    """m!(n-1-m)!/n! for m = 0..n-1 (Shapley weight of a coalition of size m
    among n players)."""
    return np.array([factorial(m) * factorial(n - 1 - m) / factorial(n) for m in range(n)])


def _path_o(tab, p, x):
    a, b = int(tab.path_offset[p]), int(tab.path_offset[p + 1])
    f = tab.feature[a + 1:b]
    lo = tab.lower[a + 1:b].astype(np.float64)
    hi = tab.upper[a + 1:b].astype(np.float64)
    xv = np.asarray(x, np.float64)[f]
    o = ((xv >= lo) & (xv < hi)).astype(np.float64)
    return f, tab.zero_fraction[a + 1:b], o


def shap_row(tab, x, n_features, n_groups):
    out = np.zeros((n_groups, n_features + 1))
    for p in range(tab.n_paths):
        f, z, o = _path_o(tab, p, x)
        k = len(f)
        g = int(tab.group[p])
        v = float(tab.v[p])
        if k == 0:
            continue
        w = _weights(k)
        for i in range(k):
            idx = [s for s in range(k) if s != i]
            c = _poly(z[idx], o[idx])
            out[g, f[i]] += v * (o[i] - z[i]) * float(np.dot(w[:len(c)], c))
    out[:, n_features] = tab.bias
    return out


def interactions_row(tab, x, n_features, n_groups):
    M1 = n_features + 1
    out = np.zeros((n_groups, M1, M1))
    shap = shap_row(tab, x, n_features, n_groups)
    for p in range(tab.n_paths):
        f, z, o = _path_o(tab, p, x)
        k = len(f)
        g = int(tab.group[p])
        v = float(tab.v[p])
        if k < 2:
            continue
        w = _weights(k - 1)
        for i in range(k):
            for j in range(k):
                if i == j:
                    continue
                idx = [s for s in range(k) if s != i and s != j]
                c = _poly(z[idx], o[idx])
                val = 0.5 * v * (o[i] - z[i]) * (o[j] - z[j]) * float(np.dot(w[:len(c)], c))
                out[g, f[i], f[j]] += val
    for g in range(n_groups):
        for i in range(n_features):
            out[g, i, i] = shap[g, i] - (out[g, i, :n_features].sum() - out[g, i, i])
        out[g, n_features, n_features] = tab.bias[g]
    return out

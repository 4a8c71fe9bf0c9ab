"""Parity bars (SURVEY.md §8(c) "Parity definitions", BASELINE.json north_star).

fp64: |got - ref| <= 1e-5 |ref| + 1e-6 for every entry, bias included.
fp32: |got - ref| <= 1e-3 max(|ref|, s_rg) for every entry, s_rg = max |ref| over
      the row-group's feature cells (normwise-relative per row and group: each
      entry sums up to ~1e6 mixed-sign contributions, so relative error near 0 is
      meaningless -- SURVEY.md §8(c)).
"""
import numpy as np


def scale(ref: np.ndarray) -> np.ndarray:
    """Per (row, group) max |ref| over feature cells (bias column/cell excluded)."""
    if ref.ndim == 3:  # phi [n][G][M+1]
        return np.abs(ref[:, :, :-1]).max(axis=2, keepdims=True) if ref.shape[2] > 1 else np.zeros(ref.shape[:2] + (1,))
    # phi_ij [n][G][M+1][M+1]
    return np.abs(ref[:, :, :-1, :-1]).max(axis=(2, 3), keepdims=True) if ref.shape[2] > 1 else np.zeros(
        ref.shape[:2] + (1, 1))


def check(got, ref, dtype: str, what: str = ""):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert got.shape == ref.shape, (got.shape, ref.shape)
    err = np.abs(got - ref)
    if dtype == "f64":
        tol = 1e-5 * np.abs(ref) + 1e-6
    else:
        tol = 1e-3 * np.maximum(np.abs(ref), scale(ref)) + 1e-9
    bad = err > tol
    if bad.any():
        idx = np.argwhere(bad)[:5]
        raise AssertionError(f"{what} parity failed ({dtype}): {int(bad.sum())} of {bad.size} entries; "
                             f"first {idx.tolist()}; got {got[tuple(idx[0])]}, ref {ref[tuple(idx[0])]}, "
                             f"max err {err.max():.3e}")
    return float(err.max())

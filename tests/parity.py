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


def check_local_accuracy(phi, f, dtype: str, what: str = ""):
    """Additivity on every row (Eq. 1 / Algorithm 1: sum_i phi_i + phi_0 = f(x)),
    normwise like the parity bar: fp32 |sum - f| <= 1e-3 s_rg + 1e-6 |f| with
    s_rg = max |phi| over the row-group's feature cells of the GPU output (one
    entry's error budget for the whole sum); fp64 1e-9 max(1, |f|)."""
    phi = np.asarray(phi, np.float64)
    f = np.asarray(f, np.float64)
    err = np.abs(phi.sum(axis=2) - f)
    if dtype == "f64":
        tol = 1e-9 * np.maximum(1.0, np.abs(f))
    else:
        tol = 1e-3 * scale(phi)[:, :, 0] + 1e-6 * np.abs(f)
    bad = err > tol
    if bad.any():
        i = np.argwhere(bad)[0]
        raise AssertionError(f"{what} local accuracy failed on {int(bad.sum())} of {bad.size} row-groups; "
                             f"first {i.tolist()}: err {err[tuple(i)]:.3e} > tol {tol[tuple(i)]:.3e}")
    return float(err.max())


def check_row_sums(phi_ij, phi, dtype: str, what: str = ""):
    """Eq. 6: the interaction matrix's rows sum to the SHAP values (feature
    cells), on every row, at the parity bar of phi (s_rg from phi)."""
    phi_ij = np.asarray(phi_ij, np.float64)
    phi = np.asarray(phi, np.float64)
    M = phi.shape[2] - 1
    got = phi_ij[:, :, :M, :M].sum(axis=3)
    ref = phi[:, :, :M]
    err = np.abs(got - ref)
    if dtype == "f64":
        tol = 1e-5 * np.abs(ref) + 1e-6
    else:
        tol = 1e-3 * np.maximum(np.abs(ref), np.abs(ref).max(axis=2, keepdims=True)) + 1e-9
    bad = err > tol
    assert not bad.any(), f"{what} row sums failed on {int(bad.sum())} entries (max err {err.max():.3e})"
    return float(err.max())


def oracle_interactions_by_trees(ens, x, parts=16, workers=4):
    """O6 on the full model, evaluated as the sum of O6 over tree subsets run
    concurrently (the values are additive over trees: PAPER.md:52, each leaf's
    contribution is separate); the bias cell of every part carries base_score,
    so (parts - 1) base_scores are taken off again.  The oracle itself is
    unchanged; this only spreads one row's ~400 core-seconds over the cores."""
    from concurrent.futures import ThreadPoolExecutor

    import oracle
    T = ens.n_trees
    cuts = [T * i // parts for i in range(parts + 1)]
    subsets = [ens.subset(range(cuts[i], cuts[i + 1])) for i in range(parts)]
    with ThreadPoolExecutor(workers) as pool:
        outs = list(pool.map(lambda e: oracle.interactions(e, x), subsets))
    total = np.sum(outs, axis=0)
    M = ens.n_features
    total[:, :, M, M] -= (parts - 1) * ens.base_score
    return total

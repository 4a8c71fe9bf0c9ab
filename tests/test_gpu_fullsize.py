"""GPU parity at BASELINE.json's full sizes (configs[2..4]), in the launch
configuration bench.py times (nodal layout, BFD packing, fp32, all rows in one
call): sampled rows against the fp64 oracle element by element, and
properties that hold at any size on every row (local accuracy against the
GPU's own bias, interaction row sums = SHAP values, symmetry)."""
import numpy as np
import pytest

import oracle
from synth.configs import WORKLOADS
from tests import parity

pytestmark = pytest.mark.gpu


def _explainer(ens, interactions=True):
    import torch
    from paper_2010_13972_b200 import TreeShapExplainer
    return TreeShapExplainer(ens, dtype="f32", pack="bfd", layout="nodal", device=torch.device("cuda:0"),
                             interactions=interactions)


def _symmetric(p):
    """phi_ij = phi_ji up to the order of the atomic adds of different blocks."""
    s = np.abs(p).max(axis=(2, 3), keepdims=True)
    return bool(np.all(np.abs(p - np.swapaxes(p, 2, 3)) <= 1e-5 * s))


def _sample(n, k, seed=0):
    """k rows spread over [0, n): both ends, tile/shard boundaries, random."""
    rng = np.random.default_rng(seed)
    edge = [0, n - 1, min(n - 1, 255), min(n - 1, 256), n // 2]
    return np.unique(np.r_[edge, rng.integers(0, n, max(0, k - len(edge)))])


def _shap_checks(name, ens, x, phi, rows):
    ref = oracle.treeshap(ens, x[rows].astype(np.float64))
    parity.check(phi[rows], ref, "f32", f"{name} sampled full-size shap")
    # the bias column is the same for every row: compare it on all rows
    np.testing.assert_allclose(phi[:, :, -1], np.broadcast_to(ref[:1, :, -1], phi[:, :, -1].shape), rtol=1e-6)


def test_adult_large_full(gpu):
    """configs[2]: 1000 trees depth 16, 14 features, 10k rows, SHAP + interactions."""
    import torch
    w = WORKLOADS["adult-large"]
    ens = w.ensemble()
    x = w.x(w.rows, ens=ens)
    ex = _explainer(ens)
    xd = torch.from_numpy(x).cuda()
    phi = ex.shap_device(xd).cpu().numpy()
    _shap_checks("adult-large", ens, x, phi, _sample(w.rows, 40))
    parity.check_local_accuracy(phi, oracle.predict(ens, x.astype(np.float64)), "f32", "adult-large")
    pij = ex.interactions_device(xd).cpu().numpy()
    rows = _sample(w.rows, 8, seed=1)
    parity.check(pij[rows], oracle.interactions(ens, x[rows].astype(np.float64)), "f32",
                 "adult-large sampled full-size interactions")
    parity.check_row_sums(pij, phi, "f32", "adult-large")
    assert _symmetric(pij)


def test_fashion_mnist_med_full_shap(gpu):
    """configs[3]: 10 classes x 100 rounds depth 8, 784 features, 10k rows (wide phi writes)."""
    import torch
    w = WORKLOADS["fashion_mnist-med"]
    ens = w.ensemble()
    x = w.x(w.rows, ens=ens)
    ex = _explainer(ens, interactions=False)
    phi = ex.shap_device(torch.from_numpy(x).cuda()).cpu().numpy()
    _shap_checks("fashion_mnist-med", ens, x, phi, _sample(w.rows, 64))
    parity.check_local_accuracy(phi, oracle.predict(ens, x.astype(np.float64)), "f32", "fashion_mnist-med")


def test_fashion_mnist_med_interactions_streamed(gpu):
    """interactions on the wide model, 24.6 MB of phi_ij per
    row, streamed in row chunks (iter_interactions) with a ragged last chunk;
    sampled rows vs the oracle, row sums vs SHAP and symmetry on every row."""
    import torch
    w = WORKLOADS["fashion_mnist-med"]
    ens = w.ensemble()
    n = 300
    x = w.x(n, ens=ens)
    ex = _explainer(ens)
    xd = torch.from_numpy(x).cuda()
    phi = ex.shap_device(xd).cpu().numpy()
    want = set(_sample(n, 6, seed=2).tolist())
    got = {}
    M = w.n_features
    for r0, r1, chunk in ex.iter_interactions(xd, chunk_rows=128):
        c = chunk.cpu().numpy()
        assert _symmetric(c), "symmetry"
        parity.check_row_sums(c, phi[r0:r1], "f32", "fashion streamed")
        for r in range(r0, r1):
            if r in want:
                got[r] = c[r - r0].astype(np.float64)
    rows = sorted(want)
    ref = oracle.interactions(ens, x[rows].astype(np.float64))
    parity.check(np.stack([got[r] for r in rows]), ref, "f32", "fashion_mnist-med streamed interactions")


def test_covtype_large_full_shap(gpu):
    """configs[4]: 8 classes x 1000 rounds depth 16, 54 features, 2^20 rows in
    one call (the bench's per-GPU shard at N=1)."""
    import torch
    w = WORKLOADS["covtype-large"]
    ens = w.ensemble()
    n = 1 << 20
    x = w.x(n, ens=ens)
    ex = _explainer(ens, interactions=False)
    phi = ex.shap_device(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.all(np.isfinite(phi))
    _shap_checks("covtype-large", ens, x, phi, _sample(n, 16))
    parity.check_local_accuracy(phi, oracle.predict(ens, x.astype(np.float64)), "f32", "covtype-large")


def test_covtype_large_full_interactions(gpu):
    """covtype interactions with the full 8000-tree model (Table 7 covtype-large
    row), 2048 rows in one call: element-wise against O6 on 4
    sampled rows (the oracle needs ~6 core-minutes per row), and on every row
    the properties that hold at any size: row sums = the SHAP kernel's values,
    symmetry, the bias cell and the zero bias row / column."""
    import torch
    w = WORKLOADS["covtype-large"]
    ens = w.ensemble()
    n = 2048
    x = w.x(n, ens=ens)
    ex = _explainer(ens)
    xd = torch.from_numpy(x).cuda()
    phi = ex.shap_device(xd).cpu().numpy()
    pij = ex.interactions_device(xd).cpu().numpy()
    M = w.n_features
    parity.check_row_sums(pij, phi, "f32", "covtype-large")
    assert _symmetric(pij)
    np.testing.assert_allclose(pij[:, :, M, M], phi[:, :, M], rtol=1e-6)
    assert np.all(pij[:, :, :M, M] == 0) and np.all(pij[:, :, M, :M] == 0)
    rows = np.array([0, 777, 1500, n - 1])
    ref = parity.oracle_interactions_by_trees(ens, x[rows].astype(np.float64))
    parity.check(pij[rows], ref, "f32", "covtype-large full-model interactions vs O6")

"""Pins for the oracle (SURVEY.md §8(c) "What pins each part").

The oracle (oracle/) is checked against things other than itself:
values the reference prints for worked examples (tests/golden/, cited),
brute-force Eq. 2 / Eq. 3-6 on small inputs, closed forms and invariants.
"""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from oracle import brute, closed_form, paths

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_fixtures.json")))


# --------------------------------------------------------------- worked examples

def test_stump_golden():
    g = GOLD["stump"]
    e = synth.stump()
    x = np.array(g["rows"])
    np.testing.assert_allclose(oracle.predict(e, x)[:, 0], g["predict"], atol=1e-15)
    np.testing.assert_allclose(oracle.treeshap(e, x[:1])[0, 0], g["phi_row0"], atol=1e-15)
    np.testing.assert_allclose(brute.shap_values(e, x[0]), g["phi_row0"], atol=1e-15)
    assert oracle.bias(e)[0] == pytest.approx(g["bias"], abs=1e-15)
    tab = paths.extract_paths(e)
    assert tab.zero_fraction[tab.feature >= 0].tolist() == pytest.approx(g["path_z"])


def test_depth2_golden():
    g = GOLD["depth2"]
    e = synth.depth2()
    x = np.array([g["row"]])
    for key, val in g["cond_expect"].items():
        assert brute.cond_expect(e, x[0], {int(c) for c in key}) == pytest.approx(val, abs=1e-15)
    np.testing.assert_allclose(oracle.treeshap(e, x)[0, 0], g["phi"], atol=1e-14)
    np.testing.assert_allclose(brute.shap_values(e, x[0]), g["phi"], atol=1e-14)
    np.testing.assert_allclose(oracle.interactions(e, x)[0, 0], g["interactions"], atol=1e-14)
    np.testing.assert_allclose(brute.interaction_values(e, x[0]), g["interactions"], atol=1e-14)
    assert np.sum(g["interactions"]) == pytest.approx(2.0)
    tab = paths.extract_paths(e)
    prods = [float(np.prod(tab.zero_fraction[tab.path_offset[p]:tab.path_offset[p + 1]]))
             for p in range(tab.n_paths)]
    assert sorted(prods) == pytest.approx(sorted(g["z_products"]))
    np.testing.assert_allclose(closed_form.shap_row(tab, x[0], 2, 1)[0], g["phi"], atol=1e-14)
    np.testing.assert_allclose(closed_form.interactions_row(tab, x[0], 2, 1)[0], g["interactions"], atol=1e-14)


def test_single_leaf_golden():
    g = GOLD["single_leaf"]
    e = synth.single_leaf(g["v"])
    np.testing.assert_allclose(oracle.treeshap(e, [[0.3]])[0, 0], g["phi"], atol=1e-15)
    np.testing.assert_allclose(oracle.interactions(e, [[0.3]])[0, 0], [[0, 0], [0, g["v"]]], atol=1e-15)


def test_extend_unwind_golden():
    g = GOLD["extend"]
    np.testing.assert_allclose(oracle.extend_chain([1, 0.4], [1, 1]), g["root_then_z04_o1"], atol=1e-15)
    np.testing.assert_allclose(oracle.extend_chain([1, 0.4], [1, 0]), g["root_then_z04_o0"], atol=1e-15)
    np.testing.assert_allclose(oracle.unwind_after_chain([1, 0.4], [1, 1], 2), g["unwind_back"], atol=1e-15)
    assert oracle.unwind_after_chain([1, 0.4], [1, 1], 2).sum() == pytest.approx(g["unwound_sum"])


# ------------------------------------------------------------ algebraic pins

def test_extend_weights_closed_form():
    """Appendix B: after root + F, w_m = [t^m] prod(z + o t) * m!(k-m)!/(k+1)!."""
    from math import factorial
    rng = np.random.default_rng(0)
    for _ in range(50):
        k = int(rng.integers(1, 10))
        z = rng.uniform(0.05, 1.0, k)
        o = rng.integers(0, 2, k).astype(float)
        w = oracle.extend_chain(np.r_[1.0, z], np.r_[1.0, o])
        c = np.array([1.0])
        for zz, oo in zip(z, o):
            c = np.convolve(c, [zz, oo])
        ref = np.array([c[m] * factorial(m) * factorial(k - m) / factorial(k + 1) for m in range(k + 1)])
        np.testing.assert_allclose(w, ref, rtol=1e-12, atol=1e-15)


def test_extend_unwind_inverse_and_commutative():
    """UNWIND undoes EXTEND for o in {0,1}, any position."""
    rng = np.random.default_rng(1)
    for _ in range(100):
        n = int(rng.integers(2, 12))
        z = np.r_[1.0, rng.uniform(0.05, 1.0, n - 1)]
        o = np.r_[1.0, rng.integers(0, 2, n - 1).astype(float)]
        i = int(rng.integers(2, n + 1))
        keep = [q for q in range(n) if q != i - 1]
        np.testing.assert_allclose(oracle.unwind_after_chain(z, o, i), oracle.extend_chain(z[keep], o[keep]),
                                   rtol=1e-9, atol=1e-12)


def _rand_ensemble(rng, max_m=6, max_t=3, max_d=5):
    M = int(rng.integers(1, max_m + 1))
    T = int(rng.integers(1, max_t + 1))
    D = int(rng.integers(1, max_d + 1))
    e = synth.make_ensemble(T, M, D, float(rng.integers(2, 2 ** D + 1)), zipf_s=float(rng.uniform(0, 2)),
                            beta=float(rng.uniform(-0.5, 0.5)), seed=int(rng.integers(1 << 30)),
                            root_cover=float(rng.integers(20, 1000)))
    e.leaf_value = rng.normal(size=e.leaf_value.shape) * (e.left < 0)
    return e


def _rand_x(rng, e, n):
    x = rng.random((n, e.n_features))
    return synth.inject_ties(x.astype(np.float32), e, 0.2, int(rng.integers(1 << 30))).astype(np.float64)


def test_treeshap_equals_eq2_bruteforce():
    """O5 (Algorithm 1 as printed) == Eq. 2 with cover weighting, incl. repeated
    features on a path and exact ties x == t (readings G1-G3)."""
    rng = np.random.default_rng(2)
    for case in range(120):
        e = _rand_ensemble(rng)
        x = _rand_x(rng, e, 3)
        phi = oracle.treeshap(e, x)
        for r in range(3):
            np.testing.assert_allclose(phi[r, 0], brute.shap_values(e, x[r]), atol=1e-12, rtol=0,
                                       err_msg=f"case {case} row {r}")


def test_interactions_equal_eq3_bruteforce():
    """O6 (conditioned on/off recursion) == Eq. 3 / Eq. 6 brute force."""
    rng = np.random.default_rng(3)
    for case in range(60):
        e = _rand_ensemble(rng, max_m=5, max_t=3, max_d=4)
        x = _rand_x(rng, e, 2)
        mat = oracle.interactions(e, x)
        for r in range(2):
            np.testing.assert_allclose(mat[r, 0], brute.interaction_values(e, x[r]), atol=1e-12, rtol=0,
                                       err_msg=f"case {case} row {r}")


def test_closed_form_equals_bruteforce_on_merged_paths():
    """O9 on the merged path table (O7) == Eq. 2/3 on the raw trees: pins the
    extraction + merge semantics and the closed form at once."""
    rng = np.random.default_rng(4)
    for case in range(60):
        e = _rand_ensemble(rng, max_m=5, max_t=2, max_d=4)
        tab = paths.extract_paths(e)
        x = _rand_x(rng, e, 2)
        for r in range(2):
            np.testing.assert_allclose(closed_form.shap_row(tab, x[r], e.n_features, 1)[0],
                                       brute.shap_values(e, x[r]), atol=1e-12)
            np.testing.assert_allclose(closed_form.interactions_row(tab, x[r], e.n_features, 1)[0],
                                       brute.interaction_values(e, x[r]), atol=1e-12)


def test_local_accuracy_and_interaction_invariants():
    """Eq. 1 additivity sum(phi)+phi_0 = f(x); interaction symmetry and row sums
    (Eq. 6), on a larger multiclass ensemble."""
    e = synth.make_ensemble(24, 9, 7, 40, n_groups=3, zipf_s=0.8, seed=11, base_score=0.25)
    x = synth.make_x(5, 64, 9).astype(np.float64)
    phi = oracle.treeshap(e, x)
    f = oracle.predict(e, x)
    np.testing.assert_allclose(phi.sum(axis=2), f, atol=1e-12)
    mat = oracle.interactions(e, x[:8])
    np.testing.assert_allclose(mat, np.swapaxes(mat, 2, 3), atol=1e-12)
    np.testing.assert_allclose(mat[:, :, :9, :9].sum(axis=3), phi[:8, :, :9], atol=1e-12)
    np.testing.assert_allclose(mat.sum(axis=(2, 3)), f[:8], atol=1e-12)


def test_unused_features_are_dummies():
    """Features never split on get phi = 0 and appending unused features changes
    nothing."""
    e = synth.make_ensemble(5, 6, 5, 20, zipf_s=3.0, seed=12)
    used = set(e.feature[e.left >= 0].tolist())
    x = synth.make_x(9, 10, 6).astype(np.float64)
    phi = oracle.treeshap(e, x)
    for f in range(6):
        if f not in used:
            assert np.all(phi[:, 0, f] == 0.0)
    wide = synth.Ensemble(e.node_offset, e.left, e.right, e.feature, e.threshold, e.cover, e.leaf_value,
                          e.tree_group, 16, 1)
    xw = np.concatenate([x, np.full((10, 10), 0.5)], axis=1)
    pw = oracle.treeshap(wide, xw)
    np.testing.assert_allclose(pw[:, 0, :6], phi[:, 0, :6], atol=1e-15)
    assert np.all(pw[:, 0, 6:16] == 0)
    iw = oracle.interactions(wide, xw[:3])
    i0 = oracle.interactions(e, x[:3])
    np.testing.assert_allclose(iw[:, 0, :6, :6], i0[:, 0, :6, :6], atol=1e-15)


def test_base_score_is_additive():
    e = synth.make_ensemble(4, 5, 4, 10, seed=13)
    e2 = synth.make_ensemble(4, 5, 4, 10, seed=13, base_score=1.5)
    x = synth.make_x(3, 5, 5).astype(np.float64)
    a, b = oracle.treeshap(e, x), oracle.treeshap(e2, x)
    np.testing.assert_allclose(b[:, :, :5], a[:, :, :5], atol=0)
    np.testing.assert_allclose(b[:, :, 5], a[:, :, 5] + 1.5, atol=1e-15)


def test_multiclass_equals_separate_groups():
    """a8: a G-group run == G single-group runs on each group's trees."""
    e = synth.make_ensemble(9, 6, 5, 16, n_groups=3, seed=14)
    x = synth.make_x(4, 12, 6).astype(np.float64)
    full = oracle.treeshap(e, x)
    for g in range(3):
        sub = e.subset([t for t in range(9) if t % 3 == g])
        sub.tree_group[:] = 0
        sub.n_groups = 1
        np.testing.assert_allclose(full[:, g], oracle.treeshap(sub, x)[:, 0], atol=1e-14)


# ------------------------------------------------------------ negative controls

def test_pins_catch_a_wrong_tie_rule():
    """Negative control: evaluating splits with x <= t (the other reading of
    PAPER.md:68) must disagree with the oracle on the tie fixture."""
    e = synth.stump()
    x_tie = np.array([[0.5]])
    assert oracle.predict(e, x_tie)[0, 0] == 0.0  # x == t goes right
    wrong = brute.shap_values(e, [np.nextafter(0.5, 0.0)])  # what x <= t would produce
    assert not np.allclose(wrong, oracle.treeshap(e, x_tie)[0, 0])


def test_pins_catch_a_dropped_half():
    """Negative control: Eq. 3 without the 1/2 (a dropped 2 in 2(M-1)!) fails the
    depth-2 golden matrix."""
    g = GOLD["depth2"]
    e = synth.depth2()
    mat = brute.interaction_values(e, g["row"])
    doubled = mat.copy()
    doubled[0, 1] *= 2
    doubled[1, 0] *= 2
    assert not np.allclose(doubled[:2, :2], np.array(g["interactions"])[:2, :2])


def test_oracle_interactions_split_over_trees():
    """The tree-partitioned evaluation the full-size GPU tests use
    (tests/parity.py: sum of O6 over tree subsets) equals one O6 call,
    base_score included."""
    from tests import parity
    ens = synth.make_ensemble(9, 6, 5, 12, n_groups=2, zipf_s=0.8, seed=41)
    ens.base_score = 0.25
    x = synth.make_x(5, 7, 6).astype(np.float64)
    np.testing.assert_allclose(parity.oracle_interactions_by_trees(ens, x, parts=4, workers=2),
                               oracle.interactions(ens, x), rtol=0, atol=1e-13)

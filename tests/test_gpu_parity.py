"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle, element by
element, on seeded inputs; plus edge cases and invariants.  Needs a B200."""
import numpy as np
import pytest

import oracle
import synth
from oracle import brute
from synth.configs import WORKLOADS
from tests import parity

pytestmark = pytest.mark.gpu

LAYOUTS = ["nodal", "warp_bins"]
DTYPES = ["f32", "f64"]


def _explainer(ens, dtype="f32", layout="nodal", pack="bfd", max_slots=0, interactions=True):
    import torch
    from paper_2010_13972_b200 import TreeShapExplainer
    return TreeShapExplainer(ens, dtype=dtype, pack=pack, layout=layout, device=torch.device("cuda:0"),
                             max_slots=max_slots, interactions=interactions)


def _run(ex, x, inter=False):
    import torch
    xd = torch.from_numpy(np.ascontiguousarray(x, dtype=ex.np_dtype)).cuda()
    out = ex.interactions_device(xd) if inter else ex.shap_device(xd)
    torch.cuda.synchronize()
    return out.cpu().numpy()


# --------------------------------------------------------------- fixtures

@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("dtype", DTYPES)
def test_spec_fixtures(gpu, layout, dtype):
    tol = 1e-12 if dtype == "f64" else 2e-6
    ex = _explainer(synth.stump(), dtype, layout)
    np.testing.assert_allclose(_run(ex, [[0.2], [0.9], [0.5]])[:, 0], [[0.6, 0.4], [-0.4, 0.4], [-0.4, 0.4]], atol=tol)
    ex = _explainer(synth.depth2(), dtype, layout)
    np.testing.assert_allclose(_run(ex, [[0.2, 0.7]])[0, 0], [1.125, 0.175, 0.7], atol=tol)
    np.testing.assert_allclose(_run(ex, [[0.2, 0.7]], inter=True)[0, 0],
                               [[1.05, 0.075, 0], [0.075, 0.1, 0], [0, 0, 0.7]], atol=tol)
    ex = _explainer(synth.single_leaf(0.7), dtype, layout)
    np.testing.assert_allclose(_run(ex, [[0.3]])[0, 0], [0.0, 0.7], atol=tol)
    np.testing.assert_allclose(_run(ex, [[0.3]], inter=True)[0, 0], [[0, 0], [0, 0.7]], atol=tol)


# ------------------------------------------------------------ config 1 (brute force)

@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("dtype", DTYPES)
def test_config1_vs_bruteforce(gpu, layout, dtype):
    w = WORKLOADS["depth3-single"]
    ens = w.ensemble()
    x = w.x(ens=ens)
    ex = _explainer(ens, dtype, layout)
    phi = _run(ex, x)
    phi_ij = _run(ex, x, inter=True)
    ref = np.stack([brute.shap_values(ens, x[r].astype(np.float64)) for r in range(len(x))])[:, None]
    ref_ij = np.stack([brute.interaction_values(ens, x[r].astype(np.float64)) for r in range(len(x))])[:, None]
    parity.check(phi, ref, dtype, "shap")
    parity.check(phi_ij, ref_ij, dtype, "interactions")
    parity.check(phi, oracle.treeshap(ens, x.astype(np.float64)), dtype, "shap vs O5")


# ------------------------------------------------------------- configs 2-5

CASES = [
    # (workload, n rows checked, n trees subset (None = all), interactions rows)
    ("cal_housing-small", 2000, None, 500),
    ("cal_housing-med", 600, None, 64),
    ("adult-large", 24, None, 4),
    ("fashion_mnist-med", 24, None, 0),
    ("covtype-large", 16, 400, 2),
]


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_configs_shap(gpu, case, dtype, layout):
    name, n, trees, _ = case
    w = WORKLOADS[name]
    ens = w.ensemble()
    if trees is not None:
        ens = ens.subset(range(trees))
    x = w.x(n, ens=ens)
    ex = _explainer(ens, dtype, layout, interactions=False)
    phi = _run(ex, x)
    ref = oracle.treeshap(ens, x.astype(np.float64))
    parity.check(phi, ref, dtype, f"{name} shap")


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("case", [c for c in CASES if c[3] > 0], ids=[c[0] for c in CASES if c[3] > 0])
def test_configs_interactions(gpu, case, dtype, layout):
    name, _, trees, n = case
    w = WORKLOADS[name]
    ens = w.ensemble()
    if trees is not None:
        ens = ens.subset(range(trees))
    x = w.x(n, ens=ens)
    ex = _explainer(ens, dtype, layout)
    got = _run(ex, x, inter=True)
    ref = oracle.interactions(ens, x.astype(np.float64))
    parity.check(got, ref, dtype, f"{name} interactions")


# ------------------------------------- skewed covers + x == t ties (wider input regime)

SKEW = [
    # (workload shape, trees kept, SHAP rows, interaction rows)
    ("cal_housing-med", 100, 400, 48),
    ("adult-large", 150, 64, 6),
    ("covtype-large", 120, 32, 4),
]


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("case", SKEW, ids=[c[0] for c in SKEW])
def test_skewed_covers_and_ties(gpu, case, dtype, layout):
    """Real GBDT covers are skewed: per-edge zero fractions from 1e-4 to
    1 - 1e-4 (synth cover_skew), where the fp32 nodal tables (rho = B/A,
    C' = v w ((1-z)/A + 1/(1-t))) and the warp-bin o = 0 UNWIND division by z
     are most exposed; plus 15 % of X entries exactly equal to a
    split threshold of their feature (x == t goes right, reading G1)."""
    import torch
    name, trees, n, ni = case
    w = WORKLOADS[name]
    ens = synth.make_ensemble(trees, w.n_features, w.max_depth, w.leaves_per_tree, n_groups=w.n_groups,
                              zipf_s=w.zipf_s, beta=w.beta, seed=w.seed + 1000, root_cover=2.0 ** 50,
                              cover_skew=1e-4)
    x = synth.inject_ties(w.x(n), ens, 0.15, seed=77)
    ex = _explainer(ens, dtype, layout)
    z = ex.paths.view()["zero_fraction"]
    assert z.min() < 2e-4 and z[z < 1].max() > 1 - 2e-4  # the skewed regime is really exercised
    x64 = x.astype(np.float64)
    parity.check(_run(ex, x), oracle.treeshap(ens, x64), dtype, f"{name} skewed shap")
    xd = torch.from_numpy(np.ascontiguousarray(x[:ni], dtype=ex.np_dtype)).cuda()
    phi, phi_ij = ex.shap_and_interactions_device(xd)
    torch.cuda.synchronize()
    parity.check(phi.cpu().numpy(), oracle.treeshap(ens, x64[:ni]), dtype, f"{name} skewed fused shap")
    parity.check(phi_ij.cpu().numpy(), oracle.interactions(ens, x64[:ni]), dtype, f"{name} skewed interactions")


# ------------------------------------------------- fused SHAP + interactions

FUSED = [c[:1] + (c[3], c[2]) for c in CASES if c[3] > 0] + [("fashion_mnist-med", 4, 120)]


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("case", FUSED, ids=[c[0] for c in FUSED])
def test_fused_shap_and_interactions(gpu, case, dtype, layout):
    """gts_shap_and_interactions: phi read off the interaction pass (NODAL) must
    match O5 and phi_ij must match O6, like the two separate calls."""
    import torch
    name, n, trees = case
    w = WORKLOADS[name]
    ens = w.ensemble()
    if trees is not None:
        ens = ens.subset(range(trees))
    x = w.x(n, ens=ens)
    ex = _explainer(ens, dtype, layout)
    xd = torch.from_numpy(np.ascontiguousarray(x, dtype=ex.np_dtype)).cuda()
    phi, phi_ij = ex.shap_and_interactions_device(xd)
    torch.cuda.synchronize()
    x64 = x.astype(np.float64)
    parity.check(phi.cpu().numpy(), oracle.treeshap(ens, x64), dtype, f"{name} fused shap")
    parity.check(phi_ij.cpu().numpy(), oracle.interactions(ens, x64), dtype, f"{name} fused interactions")


@pytest.mark.parametrize("layout", LAYOUTS)
def test_fused_ragged_and_feature_major(gpu, layout):
    import torch
    from paper_2010_13972_b200 import gts
    w = WORKLOADS["cal_housing-med"]
    ens = w.ensemble().subset(range(25))
    ex = _explainer(ens, "f32", layout)
    assert gts.gts_launches_per_call(ex.blob_int.info, 2) == (3 if layout == "nodal" else 4)
    for n in (0, 1, 33, 300):
        x = w.x(n, ens=ens)
        for fm in (False, True):
            xd = torch.from_numpy(np.ascontiguousarray(x.T)).cuda().t() if fm else torch.from_numpy(x).cuda()
            phi, phi_ij = ex.shap_and_interactions_device(xd)
            torch.cuda.synchronize()
            if n:
                x64 = x.astype(np.float64)
                parity.check(phi.cpu().numpy(), oracle.treeshap(ens, x64), "f32", f"n={n} fm={fm}")
                parity.check(phi_ij.cpu().numpy(), oracle.interactions(ens, x64), "f32", f"n={n} fm={fm} ij")


@pytest.mark.parametrize("want", ["both", "shap", "interactions"])
def test_explain_host_pipelined(gpu, want):
    """Host X -> chunked H2D / kernel / D2H on three streams -> host outputs:
    ragged last chunk, more chunks than buffer slots; parity against O5 / O6."""
    import torch
    w = WORKLOADS["cal_housing-med"]
    ens = w.ensemble().subset(range(20))
    n = 1000
    x = w.x(n, ens=ens)
    ex = _explainer(ens, "f32")
    G, M1 = ens.n_groups, ens.n_features + 1
    xh = torch.from_numpy(x).pin_memory()
    phi_h = torch.full((n, G, M1), float("nan")).pin_memory() if want != "interactions" else None
    ij_h = torch.full((n, G, M1, M1), float("nan")).pin_memory() if want != "shap" else None
    ex.explain_host_pipelined(xh, phi_h, ij_h, chunk_rows=256)
    torch.cuda.synchronize()
    x64 = x.astype(np.float64)
    if phi_h is not None:
        parity.check(phi_h.numpy(), oracle.treeshap(ens, x64), "f32", "pipelined shap")
    if ij_h is not None:
        parity.check(ij_h.numpy()[::37], oracle.interactions(ens, x64[::37]), "f32", "pipelined interactions")


@pytest.mark.parametrize("name", ["fashion_mnist-med", "covtype-large"])
def test_wide_interactions_mirror_symmetric(gpu, name):
    """Per-chunk slot maps: the kernel writes (i, j), i < j, and the mirror pass
    copies it to (j, i) over ragged 32 x 32 tiles (M+1 = 785 / 55): the result
    is exactly symmetric for every row, and matches O6 on a sample."""
    from paper_2010_13972_b200 import gts
    w = WORKLOADS[name]
    ens = w.ensemble().subset(range(60))
    x = w.x(37, ens=ens)
    ex = _explainer(ens, "f32")
    assert ex.blob_int.info.max_slots < w.n_features
    assert gts.gts_launches_per_call(ex.blob_int.info, True) == 3  # init + kernel + mirror
    got = _run(ex, x, inter=True)
    assert np.array_equal(got, np.swapaxes(got, 2, 3))
    parity.check(got[:3], oracle.interactions(ens, x[:3].astype(np.float64)), "f32", f"{name} mirror")


# ------------------------------------------------------------------ edges

@pytest.mark.parametrize("layout", LAYOUTS)
def test_ragged_rows_and_padded_ld(gpu, layout):
    import torch
    w = WORKLOADS["cal_housing-med"]
    ens = w.ensemble().subset(range(30))
    ex = _explainer(ens, "f32", layout)
    for n in (0, 1, 31, 33, 257, 1000):
        x = w.x(n, ens=ens)
        xp = np.zeros((n, 13), np.float32)
        xp[:, :8] = x
        xd = torch.from_numpy(xp).cuda()[:, :8]  # ld_x = 13 > M
        phi = ex.shap_device(xd)
        torch.cuda.synchronize()
        if n:
            parity.check(phi.cpu().numpy(), oracle.treeshap(ens, x.astype(np.float64)), "f32", f"n={n}")


def _caterpillar(depth, n_features, seed=0):
    """A chain tree of the given depth on distinct features: merged k = depth."""
    rng = np.random.default_rng(seed)
    feats = rng.permutation(n_features)[:depth]
    nodes = [None]
    cover, cur = 2.0 ** 40, 0
    for d in range(depth):
        left_c = float(np.floor(cover * rng.uniform(0.2, 0.8)))
        li, ri = len(nodes), len(nodes) + 1
        nodes += [None, {"leaf_value": float(rng.normal()), "cover": cover - left_c}]
        nodes[cur] = {"feature": int(feats[d]), "threshold": float(rng.uniform(0.3, 0.7)), "left": li, "right": ri,
                      "cover": cover}
        cur, cover = li, left_c
    nodes[cur] = {"leaf_value": float(rng.normal()), "cover": cover}
    return nodes


def _nodes_of(ens, t):
    l, r, f, th, c, v = ens.tree(t)
    return [({"leaf_value": float(v[j]), "cover": float(c[j])} if l[j] < 0 else
             {"feature": int(f[j]), "threshold": float(th[j]), "left": int(l[j]), "right": int(r[j]),
              "cover": float(c[j])}) for j in range(len(l))]


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("dtype", DTYPES)
def test_maximum_path_length(gpu, layout, dtype):
    """k = 31 distinct features on one path (merged length 32 = the warp), plus
    short paths in the same model: Q = 16 nodes, full bins."""
    trees = [_caterpillar(31, 40, seed=1), _caterpillar(20, 40, seed=2), _caterpillar(7, 40, seed=3)]
    ens = synth.ensemble_from_trees(trees, n_features=40)
    rng = np.random.default_rng(5)
    x = rng.uniform(0.25, 0.75, (64, 40)).astype(np.float32)
    ex = _explainer(ens, dtype, layout, max_slots=0 if layout == "warp_bins" else 64)
    parity.check(_run(ex, x), oracle.treeshap(ens, x.astype(np.float64)), dtype, "k=31 shap")
    parity.check(_run(ex, x[:20], inter=True), oracle.interactions(ens, x[:20].astype(np.float64)), dtype,
                 "k=31 interactions")


def _long_path_model(n_features, seed=0):
    """Chains with merged k = 31, 24 and 17 (the paper's bound is 31 features,
    PAPER.md:213-217) plus a random depth-6 forest of short paths."""
    trees = [_caterpillar(31, n_features, seed=seed + 1), _caterpillar(24, n_features, seed=seed + 2),
             _caterpillar(17, n_features, seed=seed + 3)]
    forest = synth.make_ensemble(12, n_features, 6, 30, zipf_s=0.5, seed=seed + 4)
    trees += [_nodes_of(forest, t) for t in range(forest.n_trees)]
    return synth.ensemble_from_trees(trees, n_features=n_features)


@pytest.mark.parametrize("n_features", [31, 40], ids=["identity32", "slotmaps32"])
@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("dtype", DTYPES)
def test_long_path_interactions(gpu, n_features, layout, dtype):
    """Interaction values (and the fused call) on merged paths of 17..31
    features: the default explainer builds a 32-slot interaction blob (NODAL),
    identity slot map (M = 31) or per-chunk slot maps (M = 40)."""
    import torch
    ens = _long_path_model(n_features)
    rng = np.random.default_rng(9)
    x = rng.uniform(0.2, 0.8, (70, n_features)).astype(np.float32)
    ex = _explainer(ens, dtype, layout)  # default arguments: must not fail
    if layout == "nodal":
        assert ex.blob_int.info.max_slots == 32 and ex.blob_int.info.n_tables == 3
    x64 = x.astype(np.float64)
    ref_ij = oracle.interactions(ens, x64)
    parity.check(_run(ex, x, inter=True), ref_ij, dtype, f"k<=31 interactions M={n_features}")
    parity.check(_run(ex, x), oracle.treeshap(ens, x64), dtype, f"k<=31 shap M={n_features}")
    xd = torch.from_numpy(np.ascontiguousarray(x, dtype=ex.np_dtype)).cuda()
    phi, phi_ij = ex.shap_and_interactions_device(xd[:33])
    torch.cuda.synchronize()
    parity.check(phi.cpu().numpy(), oracle.treeshap(ens, x64[:33]), dtype, "k<=31 fused shap")
    parity.check(phi_ij.cpu().numpy(), ref_ij[:33], dtype, "k<=31 fused interactions")


def test_path_too_long_rejected(gpu):
    from paper_2010_13972_b200 import gts
    ens = synth.ensemble_from_trees([_caterpillar(32, 40, seed=1)], n_features=40)
    with pytest.raises(gts.GtsError) as e:
        gts.gts_extract_paths(ens)
    assert e.value.status == 3


@pytest.mark.parametrize("layout", LAYOUTS)
def test_multiclass_base_score_single_leaves(gpu, layout):
    """G > 1, base_score, single-leaf trees (k = 0 paths only feed the bias)."""
    ens = synth.make_ensemble(30, 11, 6, 25, n_groups=3, zipf_s=1.2, seed=31)
    trees = [_nodes_of(ens, t) for t in range(ens.n_trees)] + [[{"leaf_value": 0.3, "cover": 5.0}]] * 2
    merged = synth.ensemble_from_trees(trees, n_features=11, n_groups=3, base_score=-0.75)
    x = synth.make_x(32, 300, 11)
    for dtype in DTYPES:
        ex = _explainer(merged, dtype, layout)
        parity.check(_run(ex, x), oracle.treeshap(merged, x.astype(np.float64)), dtype, "multiclass shap")
        parity.check(_run(ex, x[:40], inter=True), oracle.interactions(merged, x[:40].astype(np.float64)), dtype,
                     "multiclass interactions")


@pytest.mark.parametrize("slots", [16, 32, 64])
def test_slot_widths_and_wide_model_remap(gpu, slots):
    """Nodal blobs with every slot width; fashion-shaped M = 784 forces
    per-chunk feature remaps (slot maps) and flushes."""
    w = WORKLOADS["fashion_mnist-med"]
    ens = w.ensemble().subset(range(120))
    x = w.x(200, ens=ens)
    ex = _explainer(ens, "f32", "nodal", max_slots=slots, interactions=False)
    assert ex.blob.info.max_slots == slots
    parity.check(_run(ex, x), oracle.treeshap(ens, x.astype(np.float64)), "f32", f"slots={slots}")


@pytest.mark.parametrize("pack", ["ffd", "bfd", "nf", "none"])
def test_packing_neutrality(gpu, pack):
    """Scheduling does not change results."""
    w = WORKLOADS["cal_housing-med"]
    ens = w.ensemble()
    x = w.x(300, ens=ens)
    ex = _explainer(ens, "f64", "warp_bins", pack=pack, interactions=False)
    parity.check(_run(ex, x), oracle.treeshap(ens, x.astype(np.float64)), "f64", f"pack={pack}")


def test_local_accuracy_full_size(gpu):
    """At the bench size (cal_housing-med, 2^20 rows, the launch configuration
    bench.py times): the fused call (gts_shap_and_interactions) and the
    separate calls, element-wise against O5 / O6 on rows sampled across the
    whole range, and on every row additivity (sum phi + phi_0 = f(x)) and
    Eq. 6 row sums at the normwise bar; fused and separate results agree."""
    import torch
    w = WORKLOADS["cal_housing-med"]
    ens = w.ensemble()
    n = 1 << 20
    x = w.x(n, ens=ens)
    ex = _explainer(ens, "f32", "nodal")
    xd = torch.from_numpy(x).cuda()
    phi_f, phi_ij_f = ex.shap_and_interactions_device(xd)
    phi_f, phi_ij_f = phi_f.cpu().numpy(), phi_ij_f.cpu().numpy()
    f = oracle.predict(ens, x.astype(np.float64))
    parity.check_local_accuracy(phi_f, f, "f32", "fused 2^20")
    parity.check_row_sums(phi_ij_f, phi_f, "f32", "fused 2^20")
    rows = np.unique(np.r_[0, n - 1, np.random.default_rng(0).integers(0, n, 200)])
    x64 = x[rows].astype(np.float64)
    ref = oracle.treeshap(ens, x64)
    parity.check(phi_f[rows], ref, "f32", "sampled full-size fused shap")
    sub = rows[::6]
    ref_ij = oracle.interactions(ens, x[sub].astype(np.float64))
    parity.check(phi_ij_f[sub], ref_ij, "f32", "sampled full-size fused interactions")
    del phi_ij_f
    phi = ex.shap_device(xd).cpu().numpy()
    parity.check_local_accuracy(phi, f, "f32", "shap 2^20")
    parity.check(phi[rows], ref, "f32", "sampled full-size shap")
    parity.check(phi, phi_f.astype(np.float64), "f32", "separate vs fused shap")
    phi_ij = ex.interactions_device(xd).cpu().numpy()
    parity.check(phi_ij[sub], ref_ij, "f32", "sampled full-size interactions")
    parity.check_row_sums(phi_ij, phi, "f32", "separate 2^20")


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("name", ["cal_housing-med", "fashion_mnist-med"])
def test_feature_major_x(gpu, layout, name):
    """X given feature-major (gts_shap_strided with row_stride 1) gives the same
    results as row-major; padded column stride and a ragged row count."""
    import torch
    w = WORKLOADS[name]
    ens = w.ensemble().subset(range(60))
    n = 333
    x = w.x(n, ens=ens)
    xt = np.zeros((w.n_features, n + 7), np.float32)
    xt[:, :n] = x.T
    xd = torch.from_numpy(xt).cuda()[:, :n].t()  # shape [n][M], strides (1, n + 7)
    ex = _explainer(ens, "f32", layout, interactions=(w.n_features <= 16))
    phi = ex.shap_device(xd)
    torch.cuda.synchronize()
    parity.check(phi.cpu().numpy(), oracle.treeshap(ens, x.astype(np.float64)), "f32", "feature-major shap")
    if w.n_features <= 16:
        pij = ex.interactions_device(xd[:40])
        torch.cuda.synchronize()
        parity.check(pij.cpu().numpy(), oracle.interactions(ens, x[:40].astype(np.float64)), "f32",
                     "feature-major interactions")


@pytest.mark.parametrize("inter", [False, True])
def test_graphed_call_small_batches(gpu, inter):
    """Latency regime: the CUDA-graph replay of one call gives the oracle's
    values for new rows copied into the static buffer (1, 7 and 300 rows)."""
    w = WORKLOADS["cal_housing-small"]
    ens = w.ensemble()
    ex = _explainer(ens, "f32", "nodal")
    import torch
    for n in (1, 7, 300):
        g = ex.graphed(n, interactions=inter)
        for seed_row in (0, 5000):
            x = w.x(n, row0=seed_row, ens=ens)
            g.x.copy_(torch.from_numpy(x))
            got = g.replay().cpu().numpy()
            ref = (oracle.interactions if inter else oracle.treeshap)(ens, x.astype(np.float64))
            parity.check(got, ref, "f32", f"graphed n={n} inter={inter}")


def test_row_shards_and_replicated_blob(gpu):
    """a9: rows sharded over 4 'ranks' on one device, each with
    its own copy of the blob bytes (what the NCCL broadcast delivers), give
    the single-call result; rows on both sides of every shard boundary are
    checked against the oracle."""
    import torch
    from paper_2010_13972_b200.explainer import Blob
    w = WORKLOADS["adult-large"]
    ens = w.ensemble().subset(range(200))
    n, N = 4099, 4
    x = w.x(n, ens=ens)
    ex = _explainer(ens, "f32", "nodal")
    xd = torch.from_numpy(x).cuda()
    full = ex.shap_device(xd).cpu().numpy()
    cuts = [r * n // N for r in range(N + 1)]
    parts = []
    for r in range(N):
        rep = Blob(ex.blob.info, ex.blob.data.clone())
        out = torch.empty((cuts[r + 1] - cuts[r], 1, w.n_features + 1), device="cuda")
        from paper_2010_13972_b200 import gts
        xs = xd[cuts[r]:cuts[r + 1]]
        gts.gts_shap(rep.info, rep.ptr, xs.data_ptr(), xs.shape[0], w.n_features, out.data_ptr(),
                     torch.cuda.current_stream().cuda_stream)
        parts.append(out.cpu().numpy())
    cat = np.concatenate(parts)
    parity.check(cat, full.astype(np.float64), "f32", "shards vs single call")
    edge = sorted({c for b in cuts[1:-1] for c in (b - 1, b)})
    parity.check(cat[edge], oracle.treeshap(ens, x[edge].astype(np.float64)), "f32", "shard boundaries")


@pytest.mark.parametrize("dtype", DTYPES)
def test_validate_nonfinite_x(gpu, dtype):
    """Reading G17: gts_validate_x names the first non-finite entry (row-major
    order) for row- and feature-major X; finite X passes; the explainer's
    validate flag runs it before every call."""
    import torch
    from paper_2010_13972_b200 import gts
    w = WORKLOADS["cal_housing-med"]
    ens = w.ensemble().subset(range(10))
    ex = _explainer(ens, dtype, interactions=False)
    x = torch.from_numpy(np.ascontiguousarray(w.x(1000), dtype=ex.np_dtype)).cuda()
    ex.validate_x(x)
    ex.validate_x(x.t().contiguous().t())
    for bad in (float("nan"), float("inf"), -float("inf")):
        y = x.clone()
        y[617, 5] = bad
        y[901, 2] = bad
        for z in (y, y.t().contiguous().t()):
            with pytest.raises(gts.GtsError, match=r"X\[617\]\[5\]") as e:
                ex.validate_x(z)
            assert e.value.status == 4
    ex.validate = True
    with pytest.raises(gts.GtsError):
        ex.shap_device(y)
    ex.shap_device(x)


"""XGBoost dump_model JSON ingestion: SPEC's
examples, error classes, and a round trip of synthetic ensembles through a
dump writer (written here from the format's definition) whose parsed model
gives bit-identical path tables from the library and the oracle's SHAP values."""
import json

import numpy as np
import pytest

import oracle
from oracle import paths as opaths
from paper_2010_13972_b200 import gts
from paper_2010_13972_b200.model import DumpError, from_xgboost_dump
from synth.configs import WORKLOADS

STUMP = [{"nodeid": 0, "depth": 0, "split": "f0", "split_condition": 0.5, "yes": 1, "no": 2, "missing": 1,
          "cover": 10, "children": [{"nodeid": 1, "leaf": 1.0, "cover": 4}, {"nodeid": 2, "leaf": 0.0, "cover": 6}]}]


def _dump(ens, cover_fmt=None, hess=1.0):
    """Write an ensemble as XGBoost JSON (node ids in BFS order, as XGBoost numbers them).
    cover_fmt: None = exact; else covers are scaled by `hess` (a hessian weight),
    rounded to float32 (XGBoost's per-node stat type) and printed with this
    format (e.g. "%.6g", C++ ostream's default precision)."""
    def cv(c):
        if cover_fmt is None:
            return float(c)
        return float(cover_fmt % np.float32(c * hess))
    out = []
    for t in range(ens.n_trees):
        left, right, feat, thr, cov, val = ens.tree(t)
        ids, q = {0: 0}, [0]
        while q:
            j = q.pop(0)
            if left[j] >= 0:
                for c in (left[j], right[j]):
                    ids[int(c)] = len(ids)
                    q.append(int(c))

        def node(j):
            if left[j] < 0:
                return {"nodeid": ids[j], "leaf": float(val[j]), "cover": cv(cov[j])}
            return {"nodeid": ids[j], "split": f"f{int(feat[j])}", "split_condition": float(thr[j]),
                    "yes": ids[int(left[j])], "no": ids[int(right[j])], "missing": ids[int(left[j])],
                    "cover": cv(cov[j]), "children": [node(int(left[j])), node(int(right[j]))]}
        out.append(node(0))
    return json.dumps(out)


def test_stump_fixture():
    m = from_xgboost_dump(json.dumps(STUMP), num_class=1)
    assert m.n_trees == 1 and m.n_groups == 1 and m.n_features == 1
    assert list(m.left) == [1, -1, -1] and list(m.right) == [2, -1, -1]
    assert m.threshold[0] == np.float32(0.5) and list(m.cover) == [10, 4, 6]
    # predict cross-check against hand traversal
    assert oracle.predict(m, np.array([[0.2], [0.9]])).ravel().tolist() == [1.0, 0.0]
    # paths: stump -> z 0.4 and 0.6
    v = gts.gts_extract_paths(m).view()
    assert v["n_paths"] == 2
    np.testing.assert_array_equal(v["zero_fraction"][[1, 3]], [0.4, 0.6])


def test_round_robin_groups():
    m = from_xgboost_dump(STUMP * 4, num_class=2)
    assert m.tree_group.tolist() == [0, 1, 0, 1]


def test_errors():
    bad = json.loads(json.dumps(STUMP))
    bad[0]["split"] = "age"
    with pytest.raises(DumpError, match="f<k>"):
        from_xgboost_dump(bad)
    m = from_xgboost_dump(bad, feature_map={"age": 3})
    assert m.feature[0] == 3 and m.n_features == 4
    bad2 = json.loads(json.dumps(STUMP))
    bad2[0]["missing"] = 7
    with pytest.raises(DumpError, match="missing-branch"):
        from_xgboost_dump(bad2)
    bad3 = json.loads(json.dumps(STUMP))
    bad3[0]["yes"] = 5
    with pytest.raises(DumpError, match="dangling"):
        from_xgboost_dump(bad3)
    # cover mismatch is the library's validation
    bad4 = json.loads(json.dumps(STUMP))
    bad4[0]["children"][1]["cover"] = 7
    with pytest.raises(gts.GtsError):
        gts.gts_extract_paths(from_xgboost_dump(bad4, covers="as_is"))
    with pytest.raises(DumpError, match="cover"):
        from_xgboost_dump(bad4)


@pytest.mark.parametrize("name", ["cal_housing-med", "covtype-large"])
def test_round_trip_tables_and_values(name):
    w = WORKLOADS[name]
    ens = w.ensemble()
    if ens.n_trees > 64:
        ens = ens.subset(range(64))
    m = from_xgboost_dump(_dump(ens), num_class=w.n_groups, n_features=w.n_features)
    assert m.tree_group.tolist() == ens.tree_group.tolist()
    a, b = gts.gts_extract_paths(ens).view(), gts.gts_extract_paths(m).view()
    for k in ("path_offset", "feature", "lower", "upper", "zero_fraction", "v", "group"):
        assert np.array_equal(a[k], b[k]), k
    ref = opaths.extract_paths(m)
    assert np.array_equal(ref.zero_fraction, b["zero_fraction"])
    x = w.x(16, ens=ens).astype(np.float64)
    np.testing.assert_array_equal(oracle.treeshap(m, x), oracle.treeshap(ens, x))


@pytest.mark.parametrize("fmt", ["%.6g", "%.9g"])
def test_float32_covers_printed_at_limited_precision(fmt):
    """Real dumps: covers are float32 hessian sums printed at 6-9 significant
    digits, so parent != left + right beyond the library's 1e-6 check
    (SPEC.md:35).  covers="as_is" is rejected by the library when it does not
    conserve; "conserve" rebuilds internal covers from the leaves and the
    values move by no more than the cover rounding."""
    w = WORKLOADS["adult-large"]
    ens = w.ensemble().subset(range(40))
    doc = _dump(ens, fmt, hess=0.2371)
    raw = from_xgboost_dump(doc, n_features=w.n_features, covers="as_is")
    worst = 0.0
    for t in range(raw.n_trees):
        l, r, _, _, c, _ = raw.tree(t)
        inner = l >= 0
        worst = max(worst, float(np.max(np.abs(c[l[inner]] + c[r[inner]] - c[inner]) / c[inner])))
    if worst > 1e-6:
        with pytest.raises(gts.GtsError) as e:
            gts.gts_extract_paths(raw)
        assert e.value.status == 2
    m = from_xgboost_dump(doc, n_features=w.n_features)
    assert 0 < m.cover_adjust < 1e-5
    gts.gts_extract_paths(m)  # validates
    x = w.x(24, ens=ens).astype(np.float64)
    ref = oracle.treeshap(ens, x)
    got = oracle.treeshap(m, x)
    s = np.abs(ref[:, :, :-1]).max(axis=2, keepdims=True)
    assert np.all(np.abs(got - ref) <= 1e-4 * s + 1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("name,trees,fmt", [("covtype-large", 96, "%.6g"), ("adult-large", 60, "%.9g")])
def test_ingested_dump_through_the_kernels(gpu, name, trees, fmt):
    """An XGBoost-format dump (float32 covers printed at limited precision)
    parsed by from_xgboost_dump runs through gts_shap and the fused
    gts_shap_and_interactions call; both match O5 / O6 of the parsed model."""
    import torch

    from paper_2010_13972_b200 import TreeShapExplainer
    from tests import parity
    w = WORKLOADS[name]
    ens = w.ensemble().subset(range(trees))
    m = from_xgboost_dump(_dump(ens, fmt, hess=0.2371), num_class=w.n_groups, n_features=w.n_features)
    x = w.x(300, ens=ens)
    ex = TreeShapExplainer(m, device=torch.device("cuda:0"))
    xd = torch.from_numpy(x).cuda()
    phi = ex.shap_device(xd).cpu().numpy()
    x64 = x.astype(np.float64)
    parity.check(phi, oracle.treeshap(m, x64), "f32", f"{name} ingested shap")
    pf, pij = ex.shap_and_interactions_device(xd[:12])
    torch.cuda.synchronize()
    parity.check(pf.cpu().numpy(), oracle.treeshap(m, x64[:12]), "f32", f"{name} ingested fused shap")
    parity.check(pij.cpu().numpy(), oracle.interactions(m, x64[:12]), "f32", f"{name} ingested interactions")

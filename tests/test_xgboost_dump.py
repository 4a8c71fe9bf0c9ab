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


def _dump(ens):
    """Write an ensemble as XGBoost JSON (node ids in BFS order, as XGBoost numbers them)."""
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
                return {"nodeid": ids[j], "leaf": float(val[j]), "cover": float(cov[j])}
            return {"nodeid": ids[j], "split": f"f{int(feat[j])}", "split_condition": float(thr[j]),
                    "yes": ids[int(left[j])], "no": ids[int(right[j])], "missing": ids[int(left[j])],
                    "cover": float(cov[j]), "children": [node(int(left[j])), node(int(right[j]))]}
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
        gts.gts_extract_paths(from_xgboost_dump(bad4))


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

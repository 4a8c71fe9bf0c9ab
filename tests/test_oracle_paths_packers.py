"""Pins for the oracle's path extraction / merge (O7) and packers (O8)."""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from oracle import paths

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_fixtures.json")))
P = GOLD["packing"]


def _bins(pk):
    out = {}
    for i, b in enumerate(pk.bin_of_item.tolist()):
        out.setdefault(b, []).append(i)
    return [out[b] for b in sorted(out)]


def _check_feasible(sizes, pk, cap=32):
    fill = np.zeros(pk.n_bins, np.int64)
    lanes = {}
    for i, (b, l) in enumerate(zip(pk.bin_of_item, pk.lane_of_item)):
        fill[b] += sizes[i]
        lanes.setdefault(int(b), []).append((int(l), int(sizes[i])))
    assert np.all(fill <= cap)
    for b, ls in lanes.items():  # consecutive lanes from 0, no overlap
        ls.sort()
        pos = 0
        for l, s in ls:
            assert l == pos
            pos += s
    assert pk.sum_sizes == int(np.sum(sizes))


def test_table5_adult_small():
    """80 items of size 4 -> none 80 / 0.125, NF/FFD/BFD 10 / 1.0."""
    sizes = [4] * 80
    pk = paths.pack_none(sizes)
    assert (pk.n_bins, pk.utilisation) == (80, 0.125)
    for fn in (paths.pack_nf, paths.pack_ffd, paths.pack_bfd):
        pk = fn(sizes)
        assert (pk.n_bins, pk.utilisation) == (10, 1.0)
        _check_feasible(sizes, pk)


def test_spec_packing_traces():
    m = P["mixed"]
    assert _bins(paths.pack_nf(m["sizes"])) == m["nf_bins"]
    assert _bins(paths.pack_ffd(m["sizes"])) == m["ffd_bins"]
    assert _bins(paths.pack_bfd(m["sizes"])) == m["bfd_bins"]
    assert paths.opt_bins(m["sizes"]) == m["opt"]
    assert paths.pack_nf(P["nf_16x4"]["sizes"]).n_bins == P["nf_16x4"]["nf"]
    assert paths.pack_bfd(P["exact_fit"]["sizes"]).n_bins == P["exact_fit"]["bfd"]
    assert paths.opt_bins([1] * 32) == P["ones"]["opt"]
    assert paths.opt_bins(P["three_20"]["sizes"]) == P["three_20"]["opt"]
    with pytest.raises(ValueError):
        paths.pack_bfd([33])
    assert paths.pack_ffd([1]).utilisation == P["single_item"]["util"]


def test_ffd_bfd_differ_fixture():
    """Reading G12: hand trace on [1,5,17,17,11,8] (FFD and BFD differ only in
    assignment)."""
    s = [1, 5, 17, 17, 11, 8]
    assert paths.pack_ffd(s).bin_of_item.tolist() == [0, 1, 0, 1, 0, 1]
    assert paths.pack_bfd(s).bin_of_item.tolist() == [1, 1, 0, 1, 0, 1]


def test_ratio_bounds_vs_bruteforce_opt():
    """Table 1: K_FFD, K_BFD <= ceil(1.222 OPT)+1, K_NF <= 2 OPT."""
    rng = np.random.default_rng(0)
    for _ in range(300):
        n = int(rng.integers(1, 11))
        sizes = rng.integers(1, 33, n).tolist()
        opt = paths.opt_bins(sizes)
        for fn in (paths.pack_ffd, paths.pack_bfd):
            pk = fn(sizes)
            _check_feasible(sizes, pk)
            assert opt <= pk.n_bins <= int(np.ceil(1.222 * opt)) + 1
        nf = paths.pack_nf(sizes)
        _check_feasible(sizes, nf)
        assert nf.n_bins <= 2 * opt
        assert paths.pack_none(sizes).n_bins == n


def test_small_capacity_hook():
    """Capacities other than 32."""
    pk = paths.pack_bfd([3, 3, 2, 2, 2], capacity=4)
    _check_feasible([3, 3, 2, 2, 2], pk, cap=4)
    assert pk.n_bins == 4


# ---------------------------------------------------------------- extraction

def test_merge_examples():
    """f0 ranges (-inf,0.5) & [0.2,inf) with z .4, .5 -> [0.2,0.5), z .2;
    triple z .5 .5 .8 -> .2."""
    m = GOLD["merge"]["pair"]
    merged = paths.merge([(0, np.float32(-np.inf), np.float32(0.5), 0.4), (0, np.float32(0.2), np.float32(np.inf), 0.5)])
    assert len(merged) == 1
    f, lo, hi, z = merged[0]
    assert (float(lo), float(hi)) == (pytest.approx(m["merged_range"][0]), m["merged_range"][1])
    assert z == pytest.approx(m["merged_z"])
    t = GOLD["merge"]["triple_z"]
    merged = paths.merge([(3, -np.inf, np.inf, t["z"][0]), (3, -np.inf, np.inf, t["z"][1]), (3, -np.inf, np.inf, t["z"][2])])
    assert merged[0][3] == pytest.approx(t["merged_z"])


def test_extraction_invariants():
    """Path count = leaves; features distinct and ascending after merge, root
    first; bounds non-empty; sum v * prod z = E[f] (bias, G13); for every row and
    tree exactly one path has all o = 1 and its v is the tree's prediction
    (SPEC.md:152-157)."""
    e = synth.make_ensemble(30, 7, 8, 60, n_groups=3, zipf_s=1.5, seed=21, base_score=0.125)
    tab = paths.extract_paths(e)
    assert tab.n_paths == e.n_leaves()
    for p in range(tab.n_paths):
        a, b = tab.path_offset[p], tab.path_offset[p + 1]
        assert tab.feature[a] == -1 and tab.zero_fraction[a] == 1.0
        fs = tab.feature[a + 1:b]
        assert np.all(np.diff(fs) > 0)
        assert np.all(tab.lower[a + 1:b] < tab.upper[a + 1:b])
        assert np.all((tab.zero_fraction[a + 1:b] > 0) & (tab.zero_fraction[a + 1:b] <= 1))
    np.testing.assert_allclose(tab.bias, oracle.bias(e), rtol=1e-13)
    x = synth.make_x(22, 20, 7).astype(np.float64)
    pred = oracle.predict(e, x)
    for r in range(20):
        per_tree = {}
        for p in range(tab.n_paths):
            a, b = tab.path_offset[p], tab.path_offset[p + 1]
            f = tab.feature[a + 1:b]
            o = (x[r, f] >= tab.lower[a + 1:b]) & (x[r, f] < tab.upper[a + 1:b])
            if np.all(o):
                assert tab.tree[p] not in per_tree
                per_tree[int(tab.tree[p])] = float(tab.v[p])
        assert len(per_tree) == e.n_trees
        for g in range(3):
            s = e.base_score + sum(v for t, v in per_tree.items() if e.tree_group[t] == g)
            assert s == pytest.approx(pred[r, g], abs=1e-12)


def test_merge_idempotent():
    e = synth.make_ensemble(5, 4, 8, 50, zipf_s=2.0, seed=23)
    tab = paths.extract_paths(e)
    for p in range(tab.n_paths):
        a, b = tab.path_offset[p], tab.path_offset[p + 1]
        els = list(zip(tab.feature[a + 1:b].tolist(), tab.lower[a + 1:b], tab.upper[a + 1:b],
                       tab.zero_fraction[a + 1:b].tolist()))
        assert paths.merge(els) == els

"""Host-side hot-path steps vs the oracle, bit-exact (SURVEY.md §8(c) "Parity
definitions": path tables byte-equal to O7, bin_of_path / lane_of_path
byte-equal to O8), plus blob invariants.  CPU only."""
import os
import subprocess
import sys

import numpy as np
import pytest

import synth
from oracle import paths as op
from paper_2010_13972_b200 import gts
from synth.configs import WORKLOADS

FIELDS = ["path_offset", "feature", "lower", "upper", "zero_fraction", "v", "group", "tree", "bias"]
PACKERS = {"ffd": op.pack_ffd, "bfd": op.pack_bfd, "nf": op.pack_nf, "none": op.pack_none}


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2010_13972_b200 import _build
    _build.build()


def _same(a, b):
    return a.dtype == b.dtype and a.shape == b.shape and a.tobytes() == b.tobytes()


@pytest.mark.parametrize("name", ["depth3-single", "cal_housing-small", "cal_housing-med", "adult-large"])
def test_tables_and_packings_bit_exact(name):
    w = WORKLOADS[name]
    ens = w.ensemble()
    view = gts.gts_extract_paths(ens).view()
    ref = op.extract_paths(ens)
    for f in FIELDS:
        assert _same(view[f], getattr(ref, f)), f
    sizes = np.diff(ref.path_offset)
    p = gts.gts_extract_paths(ens)
    algos = ["ffd", "bfd", "nf", "none"] if name != "adult-large" else ["ffd", "bfd"]
    for algo in algos:
        bv = gts.gts_binpack(p, 32, algo).view()
        o = PACKERS[algo](sizes)
        assert _same(bv["bin_of_path"], o.bin_of_item) and _same(bv["lane_of_path"], o.lane_of_item), algo
        assert bv["n_bins"] == o.n_bins and bv["sum_sizes"] == o.sum_sizes
        assert bv["utilisation"] == o.sum_sizes / (32 * o.n_bins)


@pytest.mark.parametrize("name", ["fashion_mnist-med", "covtype-large"])
def test_tables_bit_exact_on_tree_samples(name):
    """Large configs: the library's full table, compared tree by tree on a
    sample of trees against the oracle's extraction of those trees."""
    w = WORKLOADS[name]
    ens = w.ensemble()
    view = gts.gts_extract_paths(ens).view()
    rng = np.random.default_rng(0)
    trees = np.sort(rng.choice(ens.n_trees, 25, replace=False))
    for t in trees:
        sub = ens.subset([t])
        ref = op.extract_paths(sub)
        sel = np.nonzero(view["tree"] == t)[0]
        assert len(sel) == ref.n_paths
        a, b = view["path_offset"][sel[0]], view["path_offset"][sel[-1] + 1]
        assert _same(view["path_offset"][sel[0]:sel[-1] + 2] - a, ref.path_offset)
        for f in ("feature", "lower", "upper", "zero_fraction"):
            assert _same(view[f][a:b], getattr(ref, f)), f
        assert _same(view["v"][sel], ref.v)
        assert np.all(view["group"][sel] == int(ens.tree_group[t]))
    import oracle
    np.testing.assert_allclose(view["bias"], oracle.bias(ens), rtol=1e-11, atol=1e-14)


def test_covtype_packing_properties():
    """6.6M items: BFD/FFD feasible, identical bin counts, within
    the Table 1 bound of the volume lower bound."""
    ens = WORKLOADS["covtype-large"].ensemble()
    p = gts.gts_extract_paths(ens)
    sizes = np.diff(p.view()["path_offset"])
    lb = int(np.ceil(sizes.sum() / 32))
    ks = {}
    for algo in ("ffd", "bfd"):
        bv = gts.gts_binpack(p, 32, algo).view()
        fill = np.bincount(bv["bin_of_path"], weights=sizes, minlength=bv["n_bins"])
        assert fill.max() <= 32 and bv["sum_sizes"] == sizes.sum()
        assert lb <= bv["n_bins"] <= int(np.ceil(1.222 * lb)) + 1
        assert bv["pack_seconds"] < 10
        ks[algo] = bv["n_bins"]
    assert ks["ffd"] == ks["bfd"]


def test_extraction_is_deterministic_across_thread_counts():
    code = ("import sys, hashlib; sys.path.insert(0, %r); from synth.configs import WORKLOADS; "
            "from paper_2010_13972_b200 import gts; v = gts.gts_extract_paths(WORKLOADS['adult-large'].ensemble()).view(); "
            "print(hashlib.sha256(b''.join(v[k].tobytes() for k in %r)).hexdigest())" % (
                os.path.dirname(os.path.dirname(os.path.abspath(__file__))), FIELDS))
    outs = set()
    for n in ("1", "3", "8"):
        env = dict(os.environ, OMP_NUM_THREADS=n)
        outs.add(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True).stdout)
    assert len(outs) == 1 and len(next(iter(outs))) > 10


def _parse_blob(blob):
    h = np.frombuffer(blob[:256].tobytes(), np.int64)
    i32 = np.frombuffer(blob[:32].tobytes(), np.int32)
    return dict(dtype=i32[2], layout=i32[3], M=i32[4], G=i32[5], S=i32[6], n_paths=h[4], n_elems=h[5], n_units=h[6],
                bytes=h[7], off_bias=h[8], off_gauss=h[9], off_units=h[10], off_work=h[11], off_slot=h[12],
                off_paths=h[13], off_elems=h[14], n_kept_paths=h[15], n_kept_elems=h[16])


CHUNK = np.dtype([("group", "i4"), ("n_paths", "i4"), ("n_slots", "i4"), ("map_id", "i4"), ("path_begin", "i8"),
                  ("elem_begin", "i8"), ("slotmap_begin", "i8"), ("n_elems", "i4"), ("table_words", "i4"),
                  ("max_q", "i4"), ("data_bytes", "i4"), ("data_off", "i8")])


@pytest.mark.parametrize("name,slots", [("cal_housing-med", 0), ("adult-large", 0), ("fashion_mnist-med", 32),
                                        ("fashion_mnist-med", 16)])
def test_nodal_blob_invariants(name, slots):
    """Every kept path (k >= 1) appears once in the staged chunk regions with
    its own feature set and nodal tables (checked against tables recomputed
    here from the oracle-independent definitions A = z + (1-z)t, B = z(1-t));
    runs share a feature set; slot maps are ascending; the Gauss rules integrate
    t^m exactly for m <= 2Q-1."""
    w = WORKLOADS[name]
    ens = w.ensemble()
    if name != "cal_housing-med":
        ens = ens.subset(range(40 if name == "adult-large" else 120))
    p = gts.gts_extract_paths(ens)
    view = p.view()
    b = gts.gts_binpack(p, 32, "bfd")
    info = gts.gts_blob_plan(b, gts.GTS_F64, "nodal", slots)
    blob = gts.gts_blob_write(b, info)
    hd = _parse_blob(blob)
    assert hd["bytes"] == info.bytes and hd["n_units"] == info.n_units
    np.testing.assert_array_equal(np.frombuffer(blob[hd["off_bias"]:hd["off_bias"] + 8 * w.n_groups].tobytes(),
                                                np.float64), view["bias"])
    g = np.frombuffer(blob[hd["off_gauss"]:hd["off_gauss"] + 8 * 16 * 3 * 16].tobytes(), np.float64).reshape(16, 3, 16)
    for Q in range(1, 17):
        t, wq = g[Q - 1, 0, :Q], g[Q - 1, 1, :Q]
        assert np.all((t > 0) & (t < 1)) and np.all(np.diff(t) > 0)
        for m in range(2 * Q):
            assert abs(np.dot(wq, t ** m) - 1.0 / (m + 1)) < 1e-14
        np.testing.assert_allclose(g[Q - 1, 2, :Q], -1.0 / (1.0 - t), rtol=1e-13)
    chunks = np.frombuffer(blob[hd["off_units"]:hd["off_units"] + 64 * hd["n_units"]].tobytes(), CHUNK)
    smap = np.frombuffer(blob[hd["off_slot"]:hd["off_elems"]].tobytes(), np.int32)
    assert info.max_chunk_bytes == chunks["data_bytes"].max() <= 16 * 1024
    # lookup of the library's own table: features -> [(v, z)]
    ref = {}
    for q in range(view["n_paths"]):
        a, bb = view["path_offset"][q] + 1, view["path_offset"][q + 1]
        if bb > a:
            ref.setdefault(tuple(view["feature"][a:bb]), []).append(
                (float(view["v"][q]), view["zero_fraction"][a:bb], view["lower"][a:bb], view["upper"][a:bb]))
    nt = 2 if hd["S"] > 16 else 3  # SHAP-only blobs drop h and alpha (blob_format.h)

    def slot_of(el):
        # element record {lo, hi, slot, w}: nt = 3 stores the slot, nt = 2 its byte offset (8-byte T here)
        return el[:, 2] if nt == 3 else el[:, 2] // 8

    seen = 0
    for c in chunks:
        n_rec = 0
        mp = smap[c["slotmap_begin"]:c["slotmap_begin"] + c["n_slots"]]
        assert np.all(np.diff(mp) > 0) and c["n_slots"] <= hd["S"]
        reg = blob[c["data_off"]:c["data_off"] + c["data_bytes"]]
        E = np.frombuffer(reg[:16 * c["n_elems"]].tobytes(), np.int32).reshape(-1, 4)
        P = np.frombuffer(reg[16 * c["n_elems"]:16 * (c["n_elems"] + c["n_paths"])].tobytes(), np.int32).reshape(-1, 4)
        tab = np.frombuffer(reg[16 * (c["n_elems"] + c["n_paths"]):].tobytes(), np.float64)
        i = 0
        while i < c["n_paths"]:
            run = P[i, 0] >> 16
            assert run >= 1
            k = P[i, 0] & 0xFF
            feats0 = tuple(mp[slot_of(E[P[i, 2]:P[i, 2] + k])])
            for j in range(run):
                kk, Q, e0, t0 = P[i + j, 0] & 0xFF, P[i + j, 1], P[i + j, 2], P[i + j, 3]
                QP = (Q + 3) & ~3
                assert kk == k and Q == (k + 1) // 2
                el = E[e0:e0 + k]
                sl = slot_of(el)
                feats = tuple(mp[sl])
                assert feats == feats0
                if nt == 3:  # slot, upper-triangle row base of the slot
                    np.testing.assert_array_equal(el[:, 3], sl * (2 * hd["S"] - sl - 1) // 2)
                else:  # slot byte offset in a tile row, the feature itself (global-X kernels)
                    np.testing.assert_array_equal(el[:, 2] % 8, 0)
                    np.testing.assert_array_equal(el[:, 3], np.array(feats))
                t, wq = g[Q - 1, 0, :Q], g[Q - 1, 1, :Q]
                d = tab[t0 + QP:t0 + QP + Q]
                v = float(-d[0] * (1 - t[0]) / wq[0])
                cands = ref[feats]
                best = min(range(len(cands)), key=lambda ii: abs(cands[ii][0] - v))
                v, z, plo, phi_ = cands.pop(best)
                A = z[:, None] + (1 - z[:, None]) * t[None]
                B = z[:, None] * (1 - t[None])
                np.testing.assert_allclose(tab[t0:t0 + Q], A.prod(axis=0), rtol=1e-12)
                np.testing.assert_allclose(tab[t0 + QP:t0 + QP + Q], -v * wq / (1 - t), rtol=1e-12, atol=1e-300)
                if nt == 3:
                    np.testing.assert_allclose(tab[t0 + 2 * QP:t0 + 2 * QP + Q], 0.5 * v * wq, rtol=1e-12, atol=1e-300)
                # element rows (blob_format.h): rho[RW] (with the bounds at BO when Q mod 4 is 1 or 2),
                # C'[QP] (, alpha[QP]); otherwise the bounds form a block of 2 x 2Q words after the path rows
                inrow = (Q & 3) in (1, 2)
                BO = (Q + 1) & ~1
                RW = (BO + 2 + 3) & ~3 if inrow else QP
                BW = 0 if inrow else 4 * Q
                ES = RW + (nt - 1) * QP
                rows = tab[t0 + nt * QP + BW:t0 + nt * QP + BW + k * ES].reshape(k, ES)
                bounds = rows[:, BO:BO + 2] if inrow else tab[t0 + nt * QP:t0 + nt * QP + 2 * k].reshape(k, 2)
                np.testing.assert_allclose(rows[:, :Q], B / A, rtol=1e-12)
                assert np.all(rows[:, Q:(BO if inrow else RW)] == 0)  # the zero pad of the node pairs
                # C' = C - d: the SHAP constant with the o = 0 share folded out (nodal.cuh shap_run)
                np.testing.assert_allclose(rows[:, RW:RW + Q], v * wq[None] * ((1 - z[:, None]) / A + 1 / (1 - t[None])),
                                           rtol=1e-12, atol=1e-300)
                if nt == 3:
                    np.testing.assert_allclose(rows[:, RW + QP:RW + QP + Q], (1 - z[:, None]) / A, rtol=1e-12, atol=1e-300)
                # the rho rows carry the path's own split bounds (as T) for EXTEND's o_s
                np.testing.assert_array_equal(bounds[:, 0], np.asarray(plo, np.float32).astype(np.float64))
                np.testing.assert_array_equal(bounds[:, 1], np.asarray(phi_, np.float32).astype(np.float64))
                # element records: the run head's (every path of a run points at them)
                assert e0 == P[i, 2]
                if j == 0:
                    n_rec += k
                seen += 1
            i += run
        assert n_rec == c["n_elems"]  # records of run heads only
    assert seen == hd["n_kept_paths"] and not any(ref.values())

"""The C ABI library (no GPU needed): loads, exports every declared symbol, and
rejects bad arguments / models with the documented status codes."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import synth
from paper_2010_13972_b200 import gts

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gts.h")


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2010_13972_b200 import _build
    _build.build()
    gts.load()


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z0-9_]+\*?\s+\*?(gts_[a-z0-9_]+)\s*\(", txt, flags=re.M)))


def test_exports_every_declared_symbol():
    names = declared_functions()
    assert len(names) >= 14
    assert sorted(names) == sorted(gts.EXPORTS)
    lib = ctypes.CDLL(gts.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    dyn = subprocess.run(["nm", "-D", "--defined-only", gts.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (gts_[a-z0-9_]+)$", dyn, flags=re.M))
    assert set(names) <= exported
    assert all(not n.startswith("gts") for n in (set(re.findall(r" T ([A-Za-z0-9_]+)$", dyn, flags=re.M)) - exported)
               if n.startswith("gts_"))


def test_version_and_status_strings():
    lib = gts.load()
    assert lib.gts_abi_version() == 4
    for code, name in gts.STATUS_NAMES.items():
        assert lib.gts_status_string(code).decode() == name


def _status(fn, *a):
    with pytest.raises(gts.GtsError) as e:
        fn(*a)
    return e.value.status


def _mut(ens, **kw):
    e = synth.Ensemble(ens.node_offset.copy(), ens.left.copy(), ens.right.copy(), ens.feature.copy(),
                       ens.threshold.copy(), ens.cover.copy(), ens.leaf_value.copy(), ens.tree_group.copy(),
                       ens.n_features, ens.n_groups, ens.base_score)
    for k, v in kw.items():
        setattr(e, k, v)
    return e


def test_invalid_models_rejected():
    base = synth.depth2()
    bad_cover = base.cover.copy(); bad_cover[3] = 2.0  # 2 + 3 != 4
    assert _status(gts.gts_extract_paths, _mut(base, cover=bad_cover)) == 2
    zero_cover = base.cover.copy(); zero_cover[2] = 0.0
    assert _status(gts.gts_extract_paths, _mut(base, cover=zero_cover)) == 2
    dangling = base.left.copy(); dangling[1] = 9
    assert _status(gts.gts_extract_paths, _mut(base, left=dangling)) == 2
    cyc = base.right.copy(); cyc[1] = 1  # child points to itself
    assert _status(gts.gts_extract_paths, _mut(base, right=cyc)) == 2
    feat = base.feature.copy(); feat[0] = 7
    assert _status(gts.gts_extract_paths, _mut(base, feature=feat)) == 2
    thr = base.threshold.copy(); thr[0] = np.nan
    assert _status(gts.gts_extract_paths, _mut(base, threshold=thr)) == 2
    grp = base.tree_group.copy(); grp[0] = 3
    assert _status(gts.gts_extract_paths, _mut(base, tree_group=grp)) == 2
    assert _status(gts.gts_extract_paths, _mut(base, n_features=0)) == 1


def test_path_too_long_and_capacity():
    # a chain of 32 distinct features: merged length 33 > 32 (reading G8)
    nodes, cover, cur = [None], float(2 ** 40), 0
    for d in range(32):
        left_c = float(np.floor(cover / 2))
        li = len(nodes)
        nodes += [None, {"leaf_value": 0.1, "cover": cover - left_c}]
        nodes[cur] = {"feature": d, "threshold": 0.5, "left": li, "right": li + 1, "cover": cover}
        cur, cover = li, left_c
    nodes[cur] = {"leaf_value": 0.2, "cover": cover}
    assert _status(gts.gts_extract_paths, synth.ensemble_from_trees([nodes], n_features=40)) == 3
    p = gts.gts_extract_paths(synth.depth2())
    assert _status(gts.gts_binpack, p, 0, "bfd") == 1
    assert _status(gts.gts_binpack, p, 33, "bfd") == 1
    assert _status(gts.gts_binpack, p, 2, "bfd") == 3  # a path of length 3 > capacity 2
    assert _status(gts.gts_binpack, p, 32, 7) == 1


def test_blob_plan_and_call_argument_errors():
    b = gts.gts_binpack(gts.gts_extract_paths(synth.depth2()), 32, "bfd")
    assert _status(gts.gts_blob_plan, b, 5, 0, 0) == 1
    assert _status(gts.gts_blob_plan, b, 0, 9, 0) == 1
    assert _status(gts.gts_blob_plan, b, 0, 0, 12) == 1
    info = gts.gts_blob_plan(b, gts.GTS_F32, "nodal")
    assert info.magic == 0x47545342 and info.abi_version == 4 and info.bytes % 256 == 0
    with pytest.raises(ValueError):
        gts.gts_blob_write(b, info, np.empty(16, np.uint8))
    # n_rows == 0 is a no-op; argument errors are caught before any CUDA call
    gts.gts_shap(info, 0, 0, 0, 2, 0)
    assert _status(gts.gts_shap, info, 16, 16, -1, 2, 16) == 1
    assert _status(gts.gts_shap, info, 16, 16, 4, 1, 16) == 1   # ld_x < n_features
    assert _status(gts.gts_shap, info, 0, 16, 4, 2, 16) == 1    # NULL blob
    assert _status(gts.gts_shap, info, 8, 16, 4, 2, 16) == 1    # misaligned blob
    bad = gts.gts_blob_info.from_bytes(info.to_bytes())
    bad.magic = 0
    assert _status(gts.gts_shap_interactions, bad, 16, 16, 4, 2, 16) == 1
    # fused call: both outputs are checked (row-major strides (2, 1))
    gts.gts_shap_and_interactions(info, 0, 0, 0, 2, 1, 0, 0)
    assert _status(gts.gts_shap_and_interactions, info, 16, 16, 4, 2, 1, 0, 16) == 1   # NULL phi
    assert _status(gts.gts_shap_and_interactions, info, 16, 16, 4, 2, 1, 16, 0) == 1   # NULL phi_ij
    assert _status(gts.gts_shap_and_interactions, info, 16, 16, 4, 2, 1, 18, 16) == 1  # misaligned phi
    assert _status(gts.gts_shap_and_interactions, bad, 16, 16, 4, 2, 1, 16, 16) == 1


def _chain(depth, n_features, seed=0):
    """One chain tree on `depth` distinct features: a merged path with k = depth."""
    rng = np.random.default_rng(seed)
    feats = rng.permutation(n_features)[:depth]
    nodes, cover, cur = [None], 2.0 ** 40, 0
    for d in range(depth):
        lc = float(np.floor(cover * 0.5))
        li, ri = len(nodes), len(nodes) + 1
        nodes += [None, {"leaf_value": 1.0, "cover": cover - lc}]
        nodes[cur] = {"feature": int(feats[d]), "threshold": 0.5, "left": li, "right": ri, "cover": cover}
        cur, cover = li, lc
    nodes[cur] = {"leaf_value": -1.0, "cover": cover}
    return nodes


def test_blob_uses_and_slot_widths():
    """gts_blob_plan_for: interaction blobs take 8/16/32 slots with 3 table rows;
    a merged path of 17..31 features needs 32; the default
    plan serves both kernels only up to 16 slots; kernels reject a blob planned
    for the other one before any launch."""
    d2 = gts.gts_binpack(gts.gts_extract_paths(synth.depth2()), 32, "bfd")
    both = gts.gts_blob_plan(d2, gts.GTS_F32, "nodal")
    assert (both.uses, both.n_tables, both.max_slots) == (gts.GTS_USE_BOTH, 3, 8)
    long_ = gts.gts_binpack(gts.gts_extract_paths(synth.ensemble_from_trees([_chain(20, 40)], n_features=40)))
    shap = gts.gts_blob_plan(long_, gts.GTS_F32, "nodal")
    assert (shap.uses, shap.n_tables, shap.max_slots) == (gts.GTS_USE_SHAP, 2, 64)
    inter = gts.gts_blob_plan_for(long_, gts.GTS_F64, "nodal", 0, "interactions")
    assert (inter.uses, inter.n_tables, inter.max_slots) == (gts.GTS_USE_INTERACTIONS, 3, 32)
    assert gts.gts_blob_write(long_, inter).nbytes == inter.bytes
    assert _status(gts.gts_blob_plan_for, long_, gts.GTS_F32, "nodal", 0, "both") == 1   # BOTH above 16 slots
    assert _status(gts.gts_blob_plan_for, long_, gts.GTS_F32, "nodal", 16, "interactions") == 1  # k = 20 > 16
    assert _status(gts.gts_blob_plan_for, long_, gts.GTS_F32, "nodal", 64, "interactions") == 1
    assert _status(gts.gts_blob_plan_for, long_, gts.GTS_F32, "nodal", 0, 7) == 1
    wide = gts.gts_binpack(gts.gts_extract_paths(synth.make_ensemble(20, 100, 6, 30, seed=3)))
    i16 = gts.gts_blob_plan_for(wide, gts.GTS_F32, "nodal", 0, "interactions")
    assert (i16.max_slots, i16.n_tables) == (16, 3)
    # wrong kernel for the blob: INVALID_ARGUMENT before anything is launched
    assert _status(gts.gts_shap_interactions, shap, 256, 256, 4, 40, 256) == 1
    assert _status(gts.gts_shap_and_interactions, shap, 256, 256, 4, 40, 1, 256, 512) == 1
    assert _status(gts.gts_shap, inter, 256, 256, 4, 40, 256) == 1
    # the write without a preceding plan re-plans from the info
    again = gts.gts_blob_info.from_bytes(inter.to_bytes())
    gts.gts_blob_plan(d2, gts.GTS_F32, "nodal")  # replaces the cached plan of d2 only
    b1 = gts.gts_blob_write(long_, again)
    gts.gts_blob_plan_for(long_, gts.GTS_F64, "nodal", 0, "interactions")
    assert np.array_equal(b1, gts.gts_blob_write(long_, inter))


def test_launch_count_and_info_roundtrip():
    b = gts.gts_binpack(gts.gts_extract_paths(synth.depth2()), 32, "bfd")
    info = gts.gts_blob_plan(b, gts.GTS_F64, "warp_bins")
    assert gts.gts_launches_per_call(info, False) == 2
    assert gts.gts_launches_per_call(info, True) == 2
    assert gts.gts_launches_per_call(info, 2) == 4  # WARP_BINS fused: both calls back to back
    nodal = gts.gts_blob_plan(b, gts.GTS_F32, "nodal")
    assert gts.gts_launches_per_call(nodal, 2) == 3  # two init fills + the interaction kernel
    again = gts.gts_blob_info.from_bytes(info.to_bytes())
    assert again.as_dict() == info.as_dict()


def test_product_path_fails_loudly_without_library(tmp_path):
    code = ("import sys; sys.path.insert(0, %r); from paper_2010_13972_b200 import gts; "
            "gts.load(%r)" % (ROOT, str(tmp_path / "missing.so")))
    r = subprocess.run(["python", "-c", code], capture_output=True, text=True)
    assert r.returncode != 0 and "native library missing" in r.stderr


@pytest.mark.parametrize("name,layout,uses", [("cal_housing-med", "nodal", "shap"), ("fashion_mnist-med", "nodal", "shap"),
                                              ("fashion_mnist-med", "nodal", "interactions"),
                                              ("cal_housing-small", "warp_bins", "shap")])
def test_blob_write_range_pieces_equal_whole(name, layout, uses):
    """gts_blob_write_range: any cut of [0, bytes) into ranges reproduces the
    bytes of gts_blob_write (head, chunk regions split mid-record, tail pad)."""
    from synth.configs import WORKLOADS
    w = WORKLOADS[name]
    ens = w.ensemble() if name != "fashion_mnist-med" else w.ensemble().subset(range(120))
    b = gts.gts_binpack(gts.gts_extract_paths(ens), 32, "bfd")
    info = gts.gts_blob_plan_for(b, gts.GTS_F32, layout, 0, uses)
    whole = gts.gts_blob_write(b, info)
    rng = np.random.default_rng(7)
    for piece in (4096, 1000, 77777, int(info.bytes)):
        got = np.full(info.bytes, 0xAB, np.uint8)
        off = 0
        while off < info.bytes:
            m = int(min(info.bytes - off, max(1, piece + rng.integers(-piece // 2, piece // 2 + 1))))
            buf = np.empty(m, np.uint8)
            gts.gts_blob_write_range(b, info, off, m, buf)
            got[off:off + m] = buf
            off += m
        assert np.array_equal(got, whole), piece
    with pytest.raises(gts.GtsError):
        gts.gts_blob_write_range(b, info, info.bytes - 4, 8, np.empty(8, np.uint8))

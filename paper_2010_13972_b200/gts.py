"""Thin ctypes binding of the C ABI in include/gts.h (argument marshalling only).

Every step of the hot path runs in the native library
(paper_2010_13972_b200/_lib/libgts.so): host C++ for extraction / packing /
blob serialisation, sm_100a kernels for the per-row work.  There is no Python
or CPU fallback: if the library is missing, loading it raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# GTS_LIB selects another in-tree build of the same sources (kernel-variant experiments)
LIB_PATH = os.environ.get("GTS_LIB") or os.path.join(_HERE, "_lib", "libgts.so")

GTS_OK = 0
STATUS_NAMES = {0: "GTS_OK", 1: "GTS_ERR_INVALID_ARGUMENT", 2: "GTS_ERR_INVALID_MODEL",
                3: "GTS_ERR_PATH_TOO_LONG", 4: "GTS_ERR_NONFINITE", 5: "GTS_ERR_CUDA",
                6: "GTS_ERR_OUT_OF_MEMORY"}
GTS_PACK_FFD, GTS_PACK_BFD, GTS_PACK_NF, GTS_PACK_NONE = 0, 1, 2, 3
PACK_ALGOS = {"ffd": 0, "bfd": 1, "nf": 2, "none": 3}
GTS_F32, GTS_F64 = 0, 1
GTS_LAYOUT_NODAL, GTS_LAYOUT_WARP_BINS = 0, 1
GTS_USE_SHAP, GTS_USE_INTERACTIONS, GTS_USE_BOTH = 1, 2, 3
USES = {"shap": 1, "interactions": 2, "both": 3}
LAYOUTS = {"nodal": 0, "warp_bins": 1}

_i64, _i32, _u32, _dbl, _vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32, ctypes.c_double, ctypes.c_void_p


class GtsError(RuntimeError):
    def __init__(self, status, message):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {message}")
        self.status = status


class gts_model(ctypes.Structure):
    _fields_ = [("n_trees", _i64), ("node_offset", _vp), ("left", _vp), ("right", _vp), ("feature", _vp),
                ("threshold", _vp), ("cover", _vp), ("leaf_value", _vp), ("tree_group", _vp),
                ("n_features", _i32), ("n_groups", _i32), ("base_score", _dbl)]


class gts_paths_view(ctypes.Structure):
    _fields_ = [("n_paths", _i64), ("n_elems", _i64), ("n_features", _i32), ("n_groups", _i32),
                ("max_len", _i32), ("path_offset", _vp), ("feature", _vp), ("lower", _vp), ("upper", _vp),
                ("zero_fraction", _vp), ("v", _vp), ("group", _vp), ("tree", _vp), ("bias", _vp)]


class gts_bins_view(ctypes.Structure):
    _fields_ = [("n_items", _i64), ("n_bins", _i64), ("sum_sizes", _i64), ("capacity", _i32), ("algo", _i32),
                ("utilisation", _dbl), ("pack_seconds", _dbl), ("bin_of_path", _vp), ("lane_of_path", _vp)]


class gts_blob_info(ctypes.Structure):
    _fields_ = [("magic", _u32), ("abi_version", _u32), ("dtype", _i32), ("layout", _i32),
                ("n_features", _i32), ("n_groups", _i32), ("max_slots", _i32), ("max_len", _i32),
                ("n_paths", _i64), ("n_elems", _i64), ("n_units", _i64), ("bytes", _i64),
                ("shap_flops_per_row", _dbl), ("inter_flops_per_row", _dbl),
                ("paper_shap_flops_per_row", _dbl), ("paper_inter_flops_per_row", _dbl),
                ("max_chunk_bytes", _i64), ("max_chunk_elems", _i64), ("max_chunk_paths", _i64),
                ("uses", _i32), ("n_tables", _i32), ("max_chunk_slots", _i32), ("chunk_bytes", _i32),
                ("reserved", _i64 * 3)]

    def to_bytes(self) -> bytes:
        return ctypes.string_at(ctypes.addressof(self), ctypes.sizeof(self))

    @classmethod
    def from_bytes(cls, b: bytes) -> "gts_blob_info":
        out = cls()
        ctypes.memmove(ctypes.addressof(out), bytes(b), ctypes.sizeof(cls))
        return out

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "reserved"}


# The symbols the header declares (checked by tests/test_abi.py).
EXPORTS = ["gts_extract_paths", "gts_paths_view_get", "gts_paths_free", "gts_binpack", "gts_bins_view_get",
           "gts_bins_free", "gts_blob_plan", "gts_blob_plan_for", "gts_blob_write", "gts_blob_write_range", "gts_shap", "gts_shap_interactions",
           "gts_shap_strided", "gts_shap_interactions_strided", "gts_shap_and_interactions",
           "gts_validate_x", "gts_launches_per_call", "gts_last_error", "gts_status_string", "gts_abi_version"]

_lib = None


def load(path: str = LIB_PATH):
    """Load libgts.so (fails loudly if it was not built: run __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"native library missing: {path} (build it with `python __graft_entry__.py` "
                          "or paper_2010_13972_b200._build.build())")
    lib = ctypes.CDLL(path)
    P = ctypes.POINTER
    lib.gts_extract_paths.argtypes = [P(gts_model), P(_vp)]
    lib.gts_paths_view_get.argtypes = [_vp, P(gts_paths_view)]
    lib.gts_paths_free.argtypes = [_vp]
    lib.gts_paths_free.restype = None
    lib.gts_binpack.argtypes = [_vp, _i32, ctypes.c_int, P(_vp)]
    lib.gts_bins_view_get.argtypes = [_vp, P(gts_bins_view)]
    lib.gts_bins_free.argtypes = [_vp]
    lib.gts_bins_free.restype = None
    lib.gts_blob_plan.argtypes = [_vp, ctypes.c_int, ctypes.c_int, _i32, P(gts_blob_info)]
    lib.gts_blob_plan_for.argtypes = [_vp, ctypes.c_int, ctypes.c_int, _i32, ctypes.c_int, P(gts_blob_info)]
    lib.gts_blob_write.argtypes = [_vp, P(gts_blob_info), _vp, ctypes.c_size_t]
    lib.gts_blob_write_range.argtypes = [_vp, P(gts_blob_info), _i64, _i64, _vp]
    for name in ("gts_shap", "gts_shap_interactions"):
        fn = getattr(lib, name)
        fn.argtypes = [P(gts_blob_info), _vp, _vp, _i64, _i64, _vp, _vp]
    for name in ("gts_shap_strided", "gts_shap_interactions_strided"):
        fn = getattr(lib, name)
        fn.argtypes = [P(gts_blob_info), _vp, _vp, _i64, _i64, _i64, _vp, _vp]
        fn.restype = ctypes.c_int
    lib.gts_shap_and_interactions.argtypes = [P(gts_blob_info), _vp, _vp, _i64, _i64, _i64, _vp, _vp, _vp]
    lib.gts_shap_and_interactions.restype = ctypes.c_int
    lib.gts_validate_x.argtypes = [ctypes.c_int, _vp, _i64, _i32, _i64, _i64, _vp]
    lib.gts_validate_x.restype = ctypes.c_int
    lib.gts_launches_per_call.argtypes = [P(gts_blob_info), _i32]
    lib.gts_launches_per_call.restype = _i32
    lib.gts_last_error.argtypes = []
    lib.gts_last_error.restype = ctypes.c_char_p
    lib.gts_status_string.argtypes = [ctypes.c_int]
    lib.gts_status_string.restype = ctypes.c_char_p
    lib.gts_abi_version.argtypes = []
    lib.gts_abi_version.restype = _i32
    for name in ("gts_extract_paths", "gts_paths_view_get", "gts_binpack", "gts_bins_view_get", "gts_blob_plan",
                 "gts_blob_plan_for",
                 "gts_blob_write", "gts_blob_write_range", "gts_shap", "gts_shap_interactions"):
        getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def _check(status):
    if status != GTS_OK:
        raise GtsError(status, (load().gts_last_error() or b"").decode())


def _arr(a, dtype):
    return np.ascontiguousarray(np.asarray(a), dtype=dtype)


def _np_view(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype)
    buf = (ctypes.c_char * (n * np.dtype(dtype).itemsize)).from_address(ptr)
    return np.frombuffer(buf, dtype=dtype, count=n).copy()


class Paths:
    """Owner of a gts_paths handle (library-owned canonical table)."""

    def __init__(self, handle, keepalive=None):
        self.handle = handle
        self._keep = keepalive

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.gts_paths_free(self.handle)
            self.handle = None

    def view(self) -> dict:
        v = gts_paths_view()
        _check(load().gts_paths_view_get(self.handle, ctypes.byref(v)))
        L, E = v.n_paths, v.n_elems
        return dict(n_paths=L, n_elems=E, n_features=v.n_features, n_groups=v.n_groups, max_len=v.max_len,
                    path_offset=_np_view(v.path_offset, L + 1, np.int64), feature=_np_view(v.feature, E, np.int32),
                    lower=_np_view(v.lower, E, np.float32), upper=_np_view(v.upper, E, np.float32),
                    zero_fraction=_np_view(v.zero_fraction, E, np.float64), v=_np_view(v.v, L, np.float64),
                    group=_np_view(v.group, L, np.int32), tree=_np_view(v.tree, L, np.int32),
                    bias=_np_view(v.bias, v.n_groups, np.float64))


class Bins:
    """Owner of a gts_bins handle."""

    def __init__(self, handle, paths):
        self.handle = handle
        self.paths = paths

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.gts_bins_free(self.handle)
            self.handle = None

    def view(self) -> dict:
        v = gts_bins_view()
        _check(load().gts_bins_view_get(self.handle, ctypes.byref(v)))
        L = v.n_items
        return dict(n_items=L, n_bins=v.n_bins, sum_sizes=v.sum_sizes, capacity=v.capacity, algo=v.algo,
                    utilisation=v.utilisation, pack_seconds=v.pack_seconds,
                    bin_of_path=_np_view(v.bin_of_path, L, np.int32),
                    lane_of_path=_np_view(v.lane_of_path, L, np.uint8))


def gts_extract_paths(model) -> Paths:
    """(1) Path extraction + duplicate merge.  ``model`` has the gts_model fields
    (node_offset, left, right, feature, threshold, cover, leaf_value,
    tree_group, n_features, n_groups, base_score)."""
    lib = load()
    keep = dict(node_offset=_arr(model.node_offset, np.int64), left=_arr(model.left, np.int32),
                right=_arr(model.right, np.int32), feature=_arr(model.feature, np.int32),
                threshold=_arr(model.threshold, np.float32), cover=_arr(model.cover, np.float64),
                leaf_value=_arr(model.leaf_value, np.float64), tree_group=_arr(model.tree_group, np.int32))
    m = gts_model(len(keep["node_offset"]) - 1, *[keep[k].ctypes.data for k in
                                                   ("node_offset", "left", "right", "feature", "threshold", "cover",
                                                    "leaf_value", "tree_group")],
                  int(model.n_features), int(model.n_groups), float(model.base_score))
    h = _vp()
    _check(lib.gts_extract_paths(ctypes.byref(m), ctypes.byref(h)))
    return Paths(h)


def gts_binpack(paths: Paths, capacity: int = 32, algo="bfd") -> Bins:
    """(2) Bin packing into warps of ``capacity`` lanes."""
    a = PACK_ALGOS[algo] if isinstance(algo, str) else int(algo)
    h = _vp()
    _check(load().gts_binpack(paths.handle, int(capacity), a, ctypes.byref(h)))
    return Bins(h, paths)


def gts_blob_plan(bins: Bins, dtype=GTS_F32, layout=GTS_LAYOUT_NODAL, max_slots: int = 0) -> gts_blob_info:
    info = gts_blob_info()
    lay = LAYOUTS[layout] if isinstance(layout, str) else int(layout)
    _check(load().gts_blob_plan(bins.handle, int(dtype), lay, int(max_slots), ctypes.byref(info)))
    return info


def gts_blob_plan_for(bins: Bins, dtype=GTS_F32, layout=GTS_LAYOUT_NODAL, max_slots: int = 0,
                      uses="both") -> gts_blob_info:
    """gts_blob_plan for an explicit use ("shap", "interactions", "both" or a GTS_USE_* value)."""
    info = gts_blob_info()
    lay = LAYOUTS[layout] if isinstance(layout, str) else int(layout)
    u = USES[uses] if isinstance(uses, str) else int(uses)
    _check(load().gts_blob_plan_for(bins.handle, int(dtype), lay, int(max_slots), u, ctypes.byref(info)))
    return info


def gts_blob_write(bins: Bins, info: gts_blob_info, dst=None) -> np.ndarray:
    """Serialise the blob into a (new or given) uint8 host array."""
    if dst is None:
        dst = np.empty(info.bytes, np.uint8)
    if dst.nbytes < info.bytes:
        raise ValueError("destination too small")
    _check(load().gts_blob_write(bins.handle, ctypes.byref(info), dst.ctypes.data, dst.nbytes))
    return dst


def gts_blob_write_range(bins: Bins, info: gts_blob_info, offset: int, nbytes: int, dst) -> None:
    """Bytes [offset, offset + nbytes) of the blob into ``dst`` (a uint8 host
    array of at least nbytes, or a raw address)."""
    ptr = dst if isinstance(dst, int) else dst.ctypes.data
    if not isinstance(dst, int) and dst.nbytes < nbytes:
        raise ValueError("destination too small")
    _check(load().gts_blob_write_range(bins.handle, ctypes.byref(info), int(offset), int(nbytes), ptr))


def gts_shap(info: gts_blob_info, d_blob: int, d_x: int, n_rows: int, ld_x: int, d_phi: int, stream: int = 0):
    """(3) SHAP values: raw device pointers (ints) and a cudaStream_t handle."""
    _check(load().gts_shap(ctypes.byref(info), d_blob, d_x, int(n_rows), int(ld_x), d_phi, stream or None))


def gts_shap_interactions(info: gts_blob_info, d_blob: int, d_x: int, n_rows: int, ld_x: int, d_phi_ij: int,
                          stream: int = 0):
    """(4) SHAP interaction values."""
    _check(load().gts_shap_interactions(ctypes.byref(info), d_blob, d_x, int(n_rows), int(ld_x), d_phi_ij,
                                        stream or None))


def gts_shap_strided(info: gts_blob_info, d_blob: int, d_x: int, n_rows: int, row_stride: int, col_stride: int,
                     d_phi: int, stream: int = 0):
    """(3) SHAP values for X[r][f] at d_x[r * row_stride + f * col_stride]."""
    _check(load().gts_shap_strided(ctypes.byref(info), d_blob, d_x, int(n_rows), int(row_stride), int(col_stride),
                                   d_phi, stream or None))


def gts_shap_interactions_strided(info: gts_blob_info, d_blob: int, d_x: int, n_rows: int, row_stride: int,
                                  col_stride: int, d_phi_ij: int, stream: int = 0):
    """(4) SHAP interaction values, strided X."""
    _check(load().gts_shap_interactions_strided(ctypes.byref(info), d_blob, d_x, int(n_rows), int(row_stride),
                                                int(col_stride), d_phi_ij, stream or None))


def gts_shap_and_interactions(info: gts_blob_info, d_blob: int, d_x: int, n_rows: int, row_stride: int,
                              col_stride: int, d_phi: int, d_phi_ij: int, stream: int = 0):
    """(3)+(4) in one pass: SHAP values and interaction values of the same rows."""
    _check(load().gts_shap_and_interactions(ctypes.byref(info), d_blob, d_x, int(n_rows), int(row_stride),
                                            int(col_stride), d_phi, d_phi_ij, stream or None))


def gts_validate_x(dtype, d_x: int, n_rows: int, n_features: int, row_stride: int, col_stride: int,
                   stream: int = 0):
    """Reading G17: raise GtsError(GTS_ERR_NONFINITE) if X holds NaN / inf (synchronises the stream)."""
    _check(load().gts_validate_x(int(dtype), d_x, int(n_rows), int(n_features), int(row_stride), int(col_stride),
                                 stream or None))


def gts_launches_per_call(info: gts_blob_info, interactions) -> int:
    """Kernel launches per call: interactions False/0 = gts_shap, True/1 = gts_shap_interactions,
    2 = gts_shap_and_interactions."""
    return int(load().gts_launches_per_call(ctypes.byref(info), int(interactions)))

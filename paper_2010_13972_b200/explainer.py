"""Public Python API: a model-bound explainer over the C ABI.

PyTorch provides device memory, streams and process groups only; every step of
the hot path runs in libgts.so.  Preprocessing (extract -> pack -> blob) runs
once per model and is amortised over all rows.
"""
from __future__ import annotations

import time

import numpy as np
import torch

from . import gts

_DT = {"f32": (gts.GTS_F32, torch.float32, np.float32), "f64": (gts.GTS_F64, torch.float64, np.float64)}


class Blob:
    """A serialised path table resident on one device (plus its host-side info)."""

    def __init__(self, info: gts.gts_blob_info, device_bytes: torch.Tensor):
        self.info = info
        self.data = device_bytes

    @property
    def ptr(self) -> int:
        return self.data.data_ptr()

    @classmethod
    def from_bins(cls, bins: gts.Bins, dtype: int, layout, max_slots: int, device) -> "Blob":
        return cls.from_info(bins, gts.gts_blob_plan(bins, dtype, layout, max_slots), device)

    STREAM_PIECE = 64 << 20  # bytes per pinned staging buffer when streaming a blob to the device

    @classmethod
    def from_info(cls, bins: gts.Bins, info: gts.gts_blob_info, device) -> "Blob":
        """Serialise the blob and place it on `device`.  Blobs larger than two
        staging pieces are streamed: range i is written on the host into one of
        two pinned buffers while range i-1 is copied H2D on a side stream, so
        the write overlaps the transfer and no blob-sized pinned buffer is
        needed (gts_blob_write_range)."""
        n = int(info.bytes)
        on_gpu = device is not None and torch.device(device).type == "cuda"
        if not on_gpu or n <= 2 * cls.STREAM_PIECE:
            host = torch.empty(n, dtype=torch.uint8, pin_memory=torch.cuda.is_available())
            gts.gts_blob_write(bins, info, host.numpy())
            dev = host.to(device, non_blocking=True) if device is not None else host
            return cls(info, dev)
        dev = torch.empty(n, dtype=torch.uint8, device=device)
        piece = cls.STREAM_PIECE
        bufs = [torch.empty(piece, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        done = [None, None]
        side = torch.cuda.Stream(device)
        for i, off in enumerate(range(0, n, piece)):
            j, m = i & 1, min(piece, n - off)
            if done[j] is not None:
                done[j].synchronize()  # the copy out of this buffer has finished
            gts.gts_blob_write_range(bins, info, off, m, bufs[j].numpy())
            with torch.cuda.stream(side):
                dev[off:off + m].copy_(bufs[j][:m], non_blocking=True)
                done[j] = torch.cuda.Event()
                done[j].record(side)
        side.synchronize()
        return cls(info, dev)

    _seq = 0  # broadcasts issued by this process (same order on every rank)

    def broadcast(self, src: int = 0, group=None) -> "Blob":
        """Replicate the source rank's blob to every rank with ONE collective:
        a broadcast of the blob bytes (NCCL over NVLink on GPUs).  The 256-byte
        info record, which the receivers need to size their buffer, goes
        through the process group's rendezvous store (host key-value plumbing,
        no device collective).  Returns self (receivers' data/info replaced)."""
        import torch.distributed as dist
        rank = dist.get_rank(group)
        Blob._seq += 1
        key = f"gts_blob_info/{Blob._seq}"
        store = _default_store()
        if store is not None:
            if rank == src:
                store.set(key, self.info.to_bytes())
            else:
                self.info = gts.gts_blob_info.from_bytes(store.get(key))
        else:  # no store reachable: the info record travels as a second, 256-byte broadcast
            dev = self.data.device
            meta = torch.zeros(256, dtype=torch.uint8, device=dev)
            if rank == src:
                raw = np.frombuffer(self.info.to_bytes(), np.uint8)
                meta[:len(raw)] = torch.from_numpy(raw.copy()).to(dev)
            dist.broadcast(meta, src, group=group)
            self.info = gts.gts_blob_info.from_bytes(meta.cpu().numpy().tobytes())
        if rank != src:
            self.data = torch.empty(self.info.bytes, dtype=torch.uint8, device=self.data.device)
        dist.broadcast(self.data, src, group=group)
        return self


def row_shard(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [floor(r n / N), floor((r+1) n / N)) of rank r; rows
    are independent, so no collective touches them."""
    return n_total * rank // world, n_total * (rank + 1) // world


def _default_store():
    try:
        from torch.distributed import distributed_c10d as c10d
        return c10d._get_default_store()
    except Exception:
        return None


class TreeShapExplainer:
    """Exact path-wise TreeShap for one tree ensemble.

    model: any object with the gts_model fields (see include/gts.h).
    dtype: "f32" (default) or "f64".  pack: "bfd" (default), "ffd", "nf", "none".
    layout: "nodal" (B200-native default) or "warp_bins" (paper lineage).
    """

    def __init__(self, model, dtype: str = "f32", pack: str = "bfd", layout: str = "nodal",
                 device=None, max_slots: int = 0, interactions: bool = True, build_blobs: bool = True,
                 inter_max_slots: int = 0, validate: bool = False, host_tables: bool = True):
        """interactions: build the interaction blob now (True) or on the first
        interaction call (False); it is never a reason to fail.  build_blobs=False
        defers both blobs (multi-GPU ranks that receive them by broadcast).
        validate: check every X for NaN / inf first (gts_validate_x, reading
        G17; costs a pass over X and a stream synchronisation).
        host_tables=False skips extraction and packing too (a rank that only
        receives blobs, see replicated())."""
        self.validate = bool(validate)
        self.dtype_code, self.torch_dtype, self.np_dtype = _DT[dtype]
        self.layout = gts.LAYOUTS[layout] if isinstance(layout, str) else int(layout)
        self.device = torch.device(device) if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else None)
        self.n_features = int(model.n_features)
        self.n_groups = int(model.n_groups)
        self.max_slots = int(max_slots)
        self.inter_max_slots = int(inter_max_slots)
        self.timings = {}
        self.paths = self.bins = None
        self._blob = self._blob_int = None
        if not host_tables:
            return
        t0 = time.perf_counter()
        self.paths = gts.gts_extract_paths(model)
        t1 = time.perf_counter()
        self.bins = gts.gts_binpack(self.paths, 32, pack)
        self.timings.update(extract_s=t1 - t0, pack_s=time.perf_counter() - t1)
        if build_blobs:
            self._blob = self._make_blob(False)
            if interactions:
                _ = self.blob_int

    def _make_blob(self, for_interactions: bool) -> Blob:
        if self.bins is None:
            raise RuntimeError("this explainer has no host tables (host_tables=False): its blobs arrive by broadcast")
        t0 = time.perf_counter()
        if self.layout == gts.GTS_LAYOUT_NODAL and for_interactions:
            info = gts.gts_blob_plan_for(self.bins, self.dtype_code, self.layout, self.inter_max_slots,
                                         "interactions")
        else:
            info = gts.gts_blob_plan(self.bins, self.dtype_code, self.layout, self.max_slots)
        t1 = time.perf_counter()
        b = Blob.from_info(self.bins, info, self.device)
        if self.device is not None and self.device.type == "cuda":
            torch.cuda.synchronize(self.device)
        k = "int_" if for_interactions else ""
        self.timings[k + "plan_s"] = t1 - t0
        self.timings[k + "write_h2d_s"] = time.perf_counter() - t1
        return b

    @classmethod
    def replicated(cls, model, mode: str = "shap", src: int = 0, group=None, **kw) -> "TreeShapExplainer":
        """Multi-GPU setup: rank `src` alone
        extracts, packs and writes the one blob `mode` needs ("shap": the SHAP
        blob; "interactions" / "both": the interaction blob, which the fused
        call also reads phi from), and ONE broadcast replicates it
        (Blob.broadcast); the other ranks do no host-side method work.  Rows
        are then sharded by the caller, with no further collectives."""
        import torch.distributed as dist
        rank = dist.get_rank(group)
        want_int = mode in ("interactions", "both")
        if rank == src:
            ex = cls(model, interactions=False, build_blobs=False, **kw)
            blob = ex.blob_int if want_int else ex.blob
        else:
            ex = cls(model, interactions=False, host_tables=False, **kw)
            blob = Blob(None, torch.empty(0, dtype=torch.uint8, device=ex.device))
        t0 = time.perf_counter()
        blob.broadcast(src, group)
        if ex.device is not None and ex.device.type == "cuda":
            torch.cuda.synchronize(ex.device)
        ex.timings["broadcast_s"] = time.perf_counter() - t0
        if want_int:
            ex._blob_int = blob
            if blob.info.uses & gts.GTS_USE_SHAP:
                ex._blob = blob
        else:
            ex._blob = blob
            if blob.info.uses & gts.GTS_USE_INTERACTIONS:
                ex._blob_int = blob
        return ex

    @property
    def blob(self) -> Blob:
        """The blob gts_shap reads (built on first use when deferred)."""
        if self._blob is None:
            self._blob = self._make_blob(False)
        return self._blob

    @blob.setter
    def blob(self, b: Blob):
        self._blob = b

    @property
    def blob_int(self) -> Blob:
        """The blob the interaction calls read: the SHAP blob itself when it
        carries the interaction tables (NODAL with <= 16 slots, WARP_BINS),
        else a blob planned for interactions (16 slots, or 32 when a merged
        path has more than 16 features)."""
        if self._blob_int is None:
            b = self._blob
            if b is not None and b.info is not None and (self.layout == gts.GTS_LAYOUT_WARP_BINS or
                                                         (b.info.uses & gts.GTS_USE_INTERACTIONS)):
                self._blob_int = b
            else:
                self._blob_int = self._make_blob(True)
        return self._blob_int

    @blob_int.setter
    def blob_int(self, b: Blob):
        self._blob_int = b

    # ------------------------------------------------------------ validation
    def _check_x(self, X) -> None:
        if not isinstance(X, torch.Tensor):
            raise TypeError("X must be a torch tensor on the explainer's device (use shap() for host arrays)")
        if X.device != self.device:
            raise ValueError(f"X is on {X.device}, the explainer on {self.device}")
        if X.dtype != self.torch_dtype:
            raise ValueError(f"X has dtype {X.dtype}, the explainer computes in {self.torch_dtype}")
        if X.dim() != 2 or X.shape[1] < self.n_features:
            raise ValueError(f"X must be [n_rows][>= {self.n_features}] (got shape {tuple(X.shape)})")
        if self.validate:
            self.validate_x(X)

    def validate_x(self, X: torch.Tensor, stream=None) -> None:
        """Raise gts.GtsError (GTS_ERR_NONFINITE) if X holds NaN or +-inf (reading G17)."""
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        rs, cs = self._strides(X)
        gts.gts_validate_x(self.dtype_code, X.data_ptr(), X.shape[0], self.n_features, rs, cs, st.cuda_stream)

    def _check_out(self, out, shape) -> None:
        if not isinstance(out, torch.Tensor) or out.device != self.device or out.dtype != self.torch_dtype:
            raise ValueError(f"out must be a {self.torch_dtype} tensor on {self.device}")
        if tuple(out.shape) != tuple(shape) or not out.is_contiguous():
            raise ValueError(f"out must be contiguous with shape {tuple(shape)} (got {tuple(out.shape)})")

    # ------------------------------------------------------------------ device
    def _device_x(self, X):
        if isinstance(X, np.ndarray):
            X = torch.from_numpy(np.ascontiguousarray(X, dtype=self.np_dtype))
        if X.dtype != self.torch_dtype:
            X = X.to(self.torch_dtype)
        if X.device != self.device:
            X = X.pin_memory().to(self.device, non_blocking=True) if X.device.type == "cpu" else X.to(self.device)
        if X.dim() != 2 or X.stride(1) != 1:
            X = X.contiguous()
        return X

    @staticmethod
    def _strides(X: torch.Tensor):
        """(row_stride, col_stride) of a row-major or feature-major [n][M] view."""
        n, m = X.shape
        if X.numel() == 0:
            return max(m, 1), 1
        if X.stride(1) == 1 or m == 1:
            return (X.stride(0) if n > 1 else m), 1
        if X.stride(0) == 1 or n == 1:
            return 1, (X.stride(1) if m > 1 else n)
        raise ValueError("X must be row-major or feature-major (one unit stride)")

    def shap_device(self, X: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """phi [n_rows][G][M+1] on the device (X already on the device, row- or feature-major)."""
        self._check_x(X)
        n = X.shape[0]
        shape = (n, self.n_groups, self.n_features + 1)
        if out is None:
            out = torch.empty(shape, dtype=self.torch_dtype, device=self.device)
        self._check_out(out, shape)
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        rs, cs = self._strides(X)
        gts.gts_shap_strided(self.blob.info, self.blob.ptr, X.data_ptr(), n, rs, cs, out.data_ptr(), st.cuda_stream)
        return out

    def interactions_device(self, X: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """phi_ij [n_rows][G][M+1][M+1] on the device."""
        self._check_x(X)
        n = X.shape[0]
        M1 = self.n_features + 1
        if out is None:
            out = torch.empty((n, self.n_groups, M1, M1), dtype=self.torch_dtype, device=self.device)
        self._check_out(out, (n, self.n_groups, M1, M1))
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        rs, cs = self._strides(X)
        gts.gts_shap_interactions_strided(self.blob_int.info, self.blob_int.ptr, X.data_ptr(), n, rs, cs,
                                          out.data_ptr(), st.cuda_stream)
        return out

    def shap_and_interactions_device(self, X: torch.Tensor, out_phi: torch.Tensor | None = None,
                                     out_phi_ij: torch.Tensor | None = None, stream=None):
        """(phi, phi_ij) of the same rows from one pass (gts_shap_and_interactions):
        the interaction kernel also writes the SHAP values, no SHAP kernel runs."""
        self._check_x(X)
        n = X.shape[0]
        M1 = self.n_features + 1
        if out_phi is None:
            out_phi = torch.empty((n, self.n_groups, M1), dtype=self.torch_dtype, device=self.device)
        if out_phi_ij is None:
            out_phi_ij = torch.empty((n, self.n_groups, M1, M1), dtype=self.torch_dtype, device=self.device)
        self._check_out(out_phi, (n, self.n_groups, M1))
        self._check_out(out_phi_ij, (n, self.n_groups, M1, M1))
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        rs, cs = self._strides(X)
        gts.gts_shap_and_interactions(self.blob_int.info, self.blob_int.ptr, X.data_ptr(), n, rs, cs,
                                      out_phi.data_ptr(), out_phi_ij.data_ptr(), st.cuda_stream)
        return out_phi, out_phi_ij

    def explain_host_pipelined(self, X_host: torch.Tensor, phi_host: torch.Tensor | None = None,
                               phi_ij_host: torch.Tensor | None = None, chunk_rows: int = 1 << 17,
                               device_budget_bytes: int = 8 << 30):
        """Host rows in, host outputs out, with the copies hidden behind the kernels.

        X_host [n][M] and the outputs (phi_host [n][G][M+1] and/or phi_ij_host
        [n][G][M+1][M+1]; None = not wanted, at least one given) should be pinned.  Rows go in
        chunks through two device buffer slots on three streams: H2D of chunk
        i+1 and D2H of chunk i-1 run while chunk i computes (gts_shap,
        gts_shap_interactions or gts_shap_and_interactions, whichever the
        outputs ask for).  Everything is ordered before the current stream,
        so the caller synchronises (or records an event) as for any other call."""
        n, M = X_host.shape
        G, M1 = self.n_groups, self.n_features + 1
        want_phi, want_ij = phi_host is not None, phi_ij_host is not None
        if not (want_phi or want_ij):
            raise ValueError("no output requested")
        if n == 0:
            return phi_host, phi_ij_host
        esz = torch.tensor([], dtype=self.torch_dtype).element_size()
        row_bytes = esz * (M + (G * M1 if want_phi else 0) + (G * M1 * M1 if want_ij else 0))
        # two device slots of cr rows each stay within device_budget_bytes
        cr = max(1, min(int(chunk_rows), n, int(device_budget_bytes) // (2 * row_bytes)))
        dev = self.device
        main = torch.cuda.current_stream(dev)
        if not hasattr(self, "_pipe_streams"):
            self._pipe_streams = tuple(torch.cuda.Stream(dev) for _ in range(3))
        hs, ks, ds = self._pipe_streams
        for st in (hs, ks, ds):
            st.wait_stream(main)
        slots = []
        for _ in range(min(2, -(-n // cr))):
            slots.append((torch.empty((cr, M), dtype=self.torch_dtype, device=dev),
                          torch.empty((cr, G, M1), dtype=self.torch_dtype, device=dev) if want_phi else None,
                          torch.empty((cr, G, M1, M1), dtype=self.torch_dtype, device=dev) if want_ij else None))
        ev_k = [None] * len(slots)
        ev_d = [None] * len(slots)
        for i, r0 in enumerate(range(0, n, cr)):
            r1 = min(n, r0 + cr)
            m = r1 - r0
            b = i % len(slots)
            xb, pb, qb = slots[b]
            if ev_k[b] is not None:
                hs.wait_event(ev_k[b])  # the kernel that read this slot's X is done
            with torch.cuda.stream(hs):
                xb[:m].copy_(X_host[r0:r1], non_blocking=True)
                e_h = torch.cuda.Event()
                e_h.record(hs)
            ks.wait_event(e_h)
            if ev_d[b] is not None:
                ks.wait_event(ev_d[b])  # this slot's outputs have reached the host
            with torch.cuda.stream(ks):
                if want_phi and want_ij:
                    self.shap_and_interactions_device(xb[:m], out_phi=pb[:m], out_phi_ij=qb[:m], stream=ks)
                elif want_phi:
                    self.shap_device(xb[:m], out=pb[:m], stream=ks)
                else:
                    self.interactions_device(xb[:m], out=qb[:m], stream=ks)
                ev_k[b] = torch.cuda.Event()
                ev_k[b].record(ks)
            ds.wait_event(ev_k[b])
            with torch.cuda.stream(ds):
                if want_phi:
                    phi_host[r0:r1].copy_(pb[:m], non_blocking=True)
                if want_ij:
                    phi_ij_host[r0:r1].copy_(qb[:m], non_blocking=True)
                ev_d[b] = torch.cuda.Event()
                ev_d[b].record(ds)
        for st in (hs, ks, ds):
            main.wait_stream(st)  # later work on the current stream (incl. reuse of the slots) waits
        return phi_host, phi_ij_host

    def graphed(self, n_rows: int, interactions: bool = False) -> "GraphedCall":
        """Latency regime: capture one call for
        a fixed row count into a CUDA graph over static X / output buffers, so
        a small batch costs one graph launch instead of two kernel launches
        plus argument checks."""
        return GraphedCall(self, n_rows, interactions)

    def interaction_bytes_per_row(self) -> int:
        return self.n_groups * (self.n_features + 1) ** 2 * torch.tensor([], dtype=self.torch_dtype).element_size()

    def iter_interactions(self, X: torch.Tensor, chunk_rows: int, stream=None, n_buffers: int = 2):
        """Row-chunked streaming of phi_ij for wide models:
        fashion_mnist-shaped models need 24.6 MB of phi_ij per row, so the rows
        are explained in chunks of `chunk_rows` into `n_buffers` rotating device
        buffers.  Yields (row0, row1, phi_ij_chunk) with the chunk's kernel
        enqueued on `stream`; a buffer is reused only after the work the caller
        enqueued on `stream` after the yield (e.g. a D2H copy or a reduction)
        has been ordered before it, since everything runs on the one stream."""
        n = X.shape[0]
        M1 = self.n_features + 1
        chunk_rows = max(1, min(int(chunk_rows), max(n, 1)))
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        bufs = [torch.empty((chunk_rows, self.n_groups, M1, M1), dtype=self.torch_dtype, device=self.device)
                for _ in range(min(n_buffers, max(1, -(-n // chunk_rows))))]
        for i, r0 in enumerate(range(0, n, chunk_rows)):
            r1 = min(n, r0 + chunk_rows)
            out = bufs[i % len(bufs)][: r1 - r0]
            self.interactions_device(X[r0:r1], out=out, stream=st)
            yield r0, r1, out

    # ------------------------------------------------------------------- host
    def shap(self, X) -> np.ndarray:
        """End to end from host X: H2D, kernels, D2H of phi."""
        Xd = self._device_x(X)
        return self.shap_device(Xd).cpu().numpy()

    def shap_interactions(self, X) -> np.ndarray:
        Xd = self._device_x(X)
        return self.interactions_device(Xd).cpu().numpy()

    def shap_and_interactions(self, X) -> tuple[np.ndarray, np.ndarray]:
        """End to end from host X: (phi, phi_ij) from one device pass."""
        Xd = self._device_x(X)
        phi, phi_ij = self.shap_and_interactions_device(Xd)
        return phi.cpu().numpy(), phi_ij.cpu().numpy()


class GraphedCall:
    """One gts_shap / gts_shap_interactions call captured in a CUDA graph.

    Copy the rows into ``x`` (static [n_rows][M] device buffer), ``replay()``,
    read ``out``.  The captured kernels are the library's own (init + main)."""

    def __init__(self, ex: TreeShapExplainer, n_rows: int, interactions: bool = False):
        self.ex = ex
        M, G = ex.n_features, ex.n_groups
        self.x = torch.zeros((n_rows, M), dtype=ex.torch_dtype, device=ex.device)
        shape = (n_rows, G, M + 1, M + 1) if interactions else (n_rows, G, M + 1)
        self.out = torch.empty(shape, dtype=ex.torch_dtype, device=ex.device)
        fn = ex.interactions_device if interactions else ex.shap_device
        side = torch.cuda.Stream(ex.device)
        side.wait_stream(torch.cuda.current_stream(ex.device))
        with torch.cuda.stream(side):  # warm-up outside capture (sets kernel attributes)
            fn(self.x, out=self.out, stream=side)
        torch.cuda.current_stream(ex.device).wait_stream(side)
        torch.cuda.synchronize(ex.device)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            fn(self.x, out=self.out, stream=torch.cuda.current_stream(ex.device))

    def replay(self) -> torch.Tensor:
        self.graph.replay()
        return self.out

"""Benchmark: exact path-wise TreeShap rows/s on B200 (SHAP + interaction
values), with roofline fraction, CPU-oracle baseline, clocks and an end-to-end
number through the public API.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload covtype-large] [--mode shap|interactions|both]
                    [--rows-per-gpu 1048576] [--rows-per-step 262144]

Default workload: BASELINE.json configs[4], covtype-large (8 classes x 1000
rounds, depth 16, 54 features) over a 2^20-row dataset per GPU, SHAP values
(PAPER.md:544 is the paper's number for this model; PAPER.md:584-601 its
row-sharded scaling).  The dataset is resident in HBM; one "step" = one
gts_shap call over the next 2^18-row window of it (windows rotate, so 4 steps
cover the 2^20 rows): a full step at 2^20 rows would take ~40 s and 25 of them
would not fit the driver's time limit.  Mode "interactions" times
gts_shap_interactions, mode "both" one gts_shap_and_interactions call (phi read
off the interaction pass; `--separate` times the two calls instead).  The
packed path table is resident (extract -> pack -> blob runs once per model,
PAPER.md:528; reported as `preprocess_ms` and in the cold `e2e_cold`).  Rows
are sharded across ranks (weak scaling); rank 0 alone builds the blob and ONE
NCCL broadcast replicates it.  At N=1 the line also carries `extra` results
for the other BASELINE configs: cal_housing-med and adult-large (mode both),
covtype-large interactions, fashion_mnist-med SHAP and interactions.  Rank 0
prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SHAP rows/sec and interaction rows/sec at 1/2/4/8 B200; % of roofline"
FP32_LANES_PER_SM = 128  # B200 (sm_100): 4 SMSP x 32 FP32 lanes
PAPER_V100 = {  # context, different hardware / model / row count
    "cal_housing-med": {"shap_rows_per_s": 111111, "interaction_rows_per_s": 5000},
    "adult-large": {"shap_rows_per_s": 2141, "interaction_rows_per_s": 72.5},
    "fashion_mnist-med": {"shap_rows_per_s": 8850, "interaction_rows_per_s": 40.7},
    "covtype-large": {"shap_rows_per_s": 196.5, "interaction_rows_per_s": 6.93},
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="covtype-large")
    ap.add_argument("--rows-per-gpu", type=int, default=1 << 20, help="rows of the resident dataset per GPU")
    ap.add_argument("--rows-per-step", type=int, default=1 << 18,
                    help="rows per timed step; steps rotate through windows of the dataset (0 = all rows)")
    ap.add_argument("--mode", choices=["both", "shap", "interactions"], default="shap")
    ap.add_argument("--extras", default="auto",
                    help="comma list workload:mode:rows timed after the main run at N=1 ('auto' = "
                         "cal_housing-med:both:1048576, adult-large:both:65536, covtype-large:interactions:4096, "
                         "fashion_mnist-med:shap:65536, fashion_mnist-med:interactions:1024; 'none')")
    ap.add_argument("--dtype", choices=["f32", "f64"], default="f32")
    ap.add_argument("--layout", choices=["nodal", "warp_bins"], default="nodal")
    ap.add_argument("--pack", default="bfd")
    ap.add_argument("--max-slots", type=int, default=0,
                    help="NODAL slot width (0 = library choice: identity map up to 64 features)")
    ap.add_argument("--x-layout", choices=["row", "feature"], default="row",
                    help="X row-major [n][M] or feature-major (gts_shap_strided, row_stride 1)")
    ap.add_argument("--phi-ij-budget-gb", type=int, default=48,
                    help="device bytes for phi_ij; larger outputs are streamed in row chunks")
    ap.add_argument("--ablation-rows", type=int, default=1 << 16)
    ap.add_argument("--pack-ablation", action="store_true",
                    help="ablation: warp-bin SHAP kernel with every packer (bfd, ffd, nf, none)")
    ap.add_argument("--latency-sweep", action="store_true",
                    help="row-count sweep 1..rows-per-gpu: eager vs CUDA-graph call latency beside the oracle")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ablation", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-serial", action="store_true",
                    help="e2e: one H2D, the call(s), one D2H, serialised (default: explain_host_pipelined)")
    ap.add_argument("--e2e-chunks", type=int, default=4,
                    help="row chunks of the pipelined e2e call (measured: 2 and 4 best, 3 and 8 lose to wave tails)")
    ap.add_argument("--separate", action="store_true",
                    help="mode both: time the step as gts_shap + gts_shap_interactions instead of the fused "
                         "gts_shap_and_interactions call")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target oracle time for cpu_baseline")
    return ap.parse_args()


# ---------------------------------------------------------------- helpers

def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ["index", "clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.active",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", self.gpu_id, "--query-gpu=" + ",".join(self.FIELDS),
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return world, rank, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ------------------------------------------------------------ CPU oracle

def cpu_oracle_rates(w, ens, mode: str, target_s: float):
    """Time the oracle (C fp64 Algorithm 1 / conditioned recursion, OpenMP over
    rows, all host cores) on a bounded sample of the workload's rows."""
    import oracle
    cores = len(os.sched_getaffinity(0))
    threads = oracle.num_threads()
    res = {}
    x_probe = w.x(64, ens=ens).astype(np.float64)
    if mode in ("both", "shap"):
        t0 = time.perf_counter()
        oracle.treeshap(ens, x_probe[:16])
        dt = max(time.perf_counter() - t0, 1e-4) / 16
        n = int(np.clip(target_s * 0.5 / dt, 16, 1 << 16))
        x = w.x(n, ens=ens).astype(np.float64)
        t0 = time.perf_counter()
        oracle.treeshap(ens, x)
        res["shap"] = (n, time.perf_counter() - t0)
    if mode in ("both", "interactions"):
        t0 = time.perf_counter()
        oracle.interactions(ens, x_probe[:4])
        dt = max(time.perf_counter() - t0, 1e-4) / 4
        n = int(np.clip(target_s * 0.5 / dt, 4, 1 << 14))
        x = w.x(n, ens=ens).astype(np.float64)
        t0 = time.perf_counter()
        oracle.interactions(ens, x)
        res["interactions"] = (n, time.perf_counter() - t0)
    sec_per_row = sum(t / n for n, t in res.values())
    sample = "; ".join(f"oracle {'O5 SHAP' if k == 'shap' else 'O6 interactions'} on the first {n} rows "
                       f"({t:.2f} s)" for k, (n, t) in res.items())
    return {"value": 1.0 / sec_per_row, "unit": "rows/s", "cores": threads, "host_cores": cores, "kind": "oracle",
            "sample": sample,
            "per_mode_rows_per_s": {k: n / t for k, (n, t) in res.items()}}


# ----------------------------------------------------------- reference arm

def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from synth.configs import WORKLOADS
    w = WORKLOADS[args.workload]
    ens = w.ensemble()
    import oracle
    oracle.build()
    # each step: a bounded sample of the workload's rows through the oracle
    per_step = max(2.0, 90.0 / max(args.steps + args.warmup, 1))
    rates, walls, sample, cores = [], [], "", 0
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        r = cpu_oracle_rates(w, ens, args.mode, per_step)
        wall = time.perf_counter() - t0
        sample, cores = r["sample"], r["cores"]
        if i >= args.warmup:
            rates.append(r["value"])
            walls.append(wall)
    v = float(np.mean(rates))
    line = {"metric": METRIC, "value": v, "unit": "rows/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 * float(np.mean(walls)), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": args.workload, "mode": args.mode, "rows_per_gpu": int(args.rows_per_gpu),
                       "global_rows": int(args.rows_per_gpu) * world, "trees": w.n_trees,
                       "max_depth": w.max_depth, "features": w.n_features, "groups": w.n_groups,
                       "note": "reference arm = the fp64 CPU oracle (oracle/treeshap.c, OpenMP over rows) on a "
                               "bounded row sample per step; rows/s combines SHAP and interaction time per row"},
            "cpu_baseline": {"value": v, "unit": "rows/s", "cores": cores, "kind": "oracle",
                             "sample": f"per step: {sample}"},
            "e2e": {"value": v, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ ours

FFMA_MEASURED_TFLOPS = 70.7  # scripts/fma_peak.cu on a B200 at 1965 MHz (profiles/r01c): scalar FFMA chains


def _windows(n: int, per_step: int):
    per = n if per_step <= 0 else min(per_step, n)
    return [(r0, min(n, r0 + per)) for r0 in range(0, n, per)]


class Runner:
    """One workload on this rank: resident X, output buffers, the timed call."""

    def __init__(self, args, w, ex, mode, n, per_step, dev, rank, separate=False):
        import torch
        self.args, self.w, self.ex, self.mode, self.n, self.dev = args, w, ex, mode, n, dev
        self.G, self.M = w.n_groups, w.n_features
        self.windows = _windows(n, per_step)
        self.rows_per_step = self.windows[0][1] - self.windows[0][0]
        self.fused = mode == "both" and not separate
        self.do_shap = mode in ("both", "shap")
        self.do_int = mode in ("both", "interactions")
        ens = w.ensemble() if w.tie_frac > 0 else None
        x_host = w.x(n, row0=rank * n, ens=ens)
        self.xh = x_host if args.dtype == "f32" else x_host.astype(np.float64)
        self.tdt = torch.float32 if args.dtype == "f32" else torch.float64
        self.esz = 4 if args.dtype == "f32" else 8
        if args.x_layout == "feature":  # [n][M] view of a feature-major [M][n] buffer
            self.xt = torch.from_numpy(np.ascontiguousarray(self.xh.T)).t()
        else:
            self.xt = torch.from_numpy(self.xh)
        self.xd = self.xt.to(dev)
        from paper_2010_13972_b200.explainer import TreeShapExplainer
        self.x_rs, self.x_cs = TreeShapExplainer._strides(self.xd)
        G, M = self.G, self.M
        W = self.rows_per_step
        self.phi = torch.empty((W, G, M + 1), dtype=self.tdt, device=dev) if self.do_shap else None
        # wide models (fashion_mnist: 24.6 MB of phi_ij per row) stream the rows in
        # chunks through one reused buffer; otherwise one call
        self.ij_row_bytes = G * (M + 1) ** 2 * self.esz
        self.ij_chunk = W if not self.do_int else max(1, min(W, (args.phi_ij_budget_gb << 30) // self.ij_row_bytes))
        self.phi_ij = (torch.empty((self.ij_chunk, G, M + 1, M + 1), dtype=self.tdt, device=dev)
                       if self.do_int else None)
        self.stream = torch.cuda.current_stream(dev)

    def call(self, i, evs=None):
        """Step i: the hot path over window i mod n_windows; evs[0]/evs[1] bracket it."""
        from paper_2010_13972_b200 import gts
        r0, r1 = self.windows[i % len(self.windows)]
        ex, st = self.ex, self.stream.cuda_stream
        if evs:
            evs[0].record(self.stream)
        if self.fused:
            for c0 in range(r0, r1, self.ij_chunk):
                c1 = min(r1, c0 + self.ij_chunk)
                xr = self.xd[c0:c1]
                gts.gts_shap_and_interactions(ex.blob_int.info, ex.blob_int.ptr, xr.data_ptr(), c1 - c0, self.x_rs,
                                              self.x_cs, self.phi[c0 - r0:c1 - r0].data_ptr(), self.phi_ij.data_ptr(),
                                              st)
        else:
            if self.do_shap:
                xr = self.xd[r0:r1]
                gts.gts_shap_strided(ex.blob.info, ex.blob.ptr, xr.data_ptr(), r1 - r0, self.x_rs, self.x_cs,
                                     self.phi.data_ptr(), st)
            if self.do_int:
                for c0 in range(r0, r1, self.ij_chunk):
                    c1 = min(r1, c0 + self.ij_chunk)
                    xr = self.xd[c0:c1]
                    gts.gts_shap_interactions_strided(ex.blob_int.info, ex.blob_int.ptr, xr.data_ptr(), c1 - c0,
                                                      self.x_rs, self.x_cs, self.phi_ij.data_ptr(), st)
        if evs:
            evs[1].record(self.stream)
        return r1 - r0

    def launches_per_step(self):
        from paper_2010_13972_b200 import gts
        n_chunks = -(-self.rows_per_step // self.ij_chunk)
        if self.fused:
            return gts.gts_launches_per_call(self.ex.blob_int.info, 2) * n_chunks
        return ((gts.gts_launches_per_call(self.ex.blob.info, False) if self.do_shap else 0) +
                (gts.gts_launches_per_call(self.ex.blob_int.info, True) * n_chunks if self.do_int else 0))

    def timed(self, steps, warmup, flush, world, clk=None):
        """W untimed + K timed steps (L2 flushed before each, outside the events);
        returns per-step device ms (CUDA events on the launch stream) and rows."""
        import torch
        for i in range(warmup):
            self.call(i)
        torch.cuda.synchronize()
        barrier(world)
        torch.cuda.synchronize()
        ms, rows = [], []
        for i in range(steps):
            flush.zero_()
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            rows.append(self.call(warmup + i, evs))
            torch.cuda.synchronize()
            ms.append(evs[0].elapsed_time(evs[1]))
        torch.cuda.synchronize()
        barrier(world)
        return ms, rows

    def flops_per_row(self):
        if self.mode == "shap":
            info = self.ex.blob.info
            return info.shap_flops_per_row, info.paper_shap_flops_per_row
        info = self.ex.blob_int.info
        return info.inter_flops_per_row, info.paper_inter_flops_per_row


def roofline(flops_per_row, paper_flops_per_row, rows, ms, peak, f_med_over_max):
    """Dominant kernel's roofline: FP32-ALU bound; achieved =
    algorithmic flops per launch / event time.  frac_nodal counts what the
    nodal formulation computes (gts_blob_info.*_flops_per_row, DESIGN R1);
    frac_survey_8d counts SURVEY §8(d)'s op count of the paper's recurrence
    (it exceeds 1 when the nodal form needs fewer operations)."""
    if ms <= 0:
        return None
    ach = flops_per_row * rows / (ms / 1000.0) / 1e12
    paper = paper_flops_per_row * rows / (ms / 1000.0) / 1e12
    return {"bound": "alu", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
            "frac_nodal": ach / peak, "frac_survey_8d": paper / peak,
            "peak_kind": "nominal: SMs x 128 FP32 lanes x 2 x max SM clock",
            "peak_ffma_measured": FFMA_MEASURED_TFLOPS, "frac_vs_ffma_measured": ach / FFMA_MEASURED_TFLOPS,
            "frac_at_median_clock": ach / (peak * f_med_over_max), "traffic": None,
            "flops_per_row": flops_per_row, "paper_flops_per_row": paper_flops_per_row,
            "survey_8d_equiv_tflops": paper}


def _traffic_entry(workload, layout, mode, dtype):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return json.load(open(path)).get(f"{workload}/{layout}/{mode}/{dtype}")
    except Exception:
        return None


def run_ours(args):
    import torch

    from paper_2010_13972_b200.explainer import TreeShapExplainer
    from synth.configs import WORKLOADS

    world, rank, local = dist_setup(args)
    dev = torch.device("cuda", local)
    w = WORKLOADS[args.workload]
    ens = w.ensemble()
    M, G = w.n_features, w.n_groups
    n = int(args.rows_per_gpu)
    mode = args.mode
    fused = mode == "both" and not args.separate
    kw = dict(dtype=args.dtype, pack=args.pack, layout=args.layout, device=dev, max_slots=args.max_slots)

    # --- model preprocessing: rank 0 extracts + packs + writes the blob the mode
    #     needs; ONE broadcast replicates it (TreeShapExplainer.replicated)
    t0 = time.perf_counter()
    if world > 1:
        barrier(world)
        ex = TreeShapExplainer.replicated(ens, mode=("both" if fused else mode) if not args.separate else mode,
                                          **kw)
        if args.separate and mode == "both":
            _ = ex.blob  # --separate needs the SHAP blob too (not part of the one-broadcast setup)
    else:
        ex = TreeShapExplainer(ens, interactions=False, build_blobs=False, **kw)
        if mode in ("shap",) or (mode == "both" and args.separate):
            _ = ex.blob
        if mode in ("interactions", "both"):
            _ = ex.blob_int
    torch.cuda.synchronize()
    pre_ms = 1000 * (time.perf_counter() - t0)
    timings = dict(ex.timings)
    bcast_ms = 1000 * timings.get("broadcast_s", 0.0)
    info_main = ex.blob.info if mode == "shap" else ex.blob_int.info
    bins_view = ex.bins.view() if ex.bins is not None else None

    run = Runner(args, w, ex, mode, n, args.rows_per_step, dev, rank, separate=args.separate)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    gpu_uuid = str(torch.cuda.get_device_properties(dev).uuid)
    gpu_id = gpu_uuid if gpu_uuid.startswith("GPU-") else "GPU-" + gpu_uuid
    with ClockSampler(gpu_id) as clk:
        ms, rows = run.timed(args.steps, args.warmup, flush, world)
    clocks = clk.summary()
    ms_step = max_over_ranks(float(np.mean(ms)), world)
    ms_med = max_over_ranks(float(np.median(ms)), world)
    ms_min = max_over_ranks(float(np.min(ms)), world)
    rows_step = int(np.mean(rows))

    # --- end to end through the public API: pinned host X -> device -> host outputs
    e2e = e2e_cold = None
    if not args.no_e2e:
        W = run.rows_per_step
        x_pin = run.xt.pin_memory()  # the whole dataset: every window's H2D reads pinned memory
        phi_h = torch.empty((W, G, M + 1), dtype=run.tdt, pin_memory=True) if run.do_shap else None
        phi_ij_h = None
        pipelined = not args.e2e_serial and run.ij_chunk == W and args.x_layout == "row"
        if run.do_int:
            rows_h = W if pipelined else run.ij_chunk
            phi_ij_h = torch.empty((min(rows_h, max(1, (4 << 30) // run.ij_row_bytes)), G, M + 1, M + 1),
                                   dtype=run.tdt, pin_memory=True)
            if phi_ij_h.shape[0] < W:
                pipelined = False
        if pipelined and run.phi_ij is not None:
            run.phi_ij = None  # the pipelined call has its own device slots
            torch.cuda.empty_cache()
        xe = torch.empty((W, run.xd.shape[1]), dtype=run.tdt, device=dev)
        stream = run.stream

        def e2e_step(i):
            r0, r1 = run.windows[i % len(run.windows)]
            m = r1 - r0
            if pipelined:
                ex.explain_host_pipelined(x_pin[r0:r1], phi_h[:m] if run.do_shap else None,
                                          phi_ij_h[:m] if run.do_int else None,
                                          chunk_rows=max(1, -(-m // args.e2e_chunks)))
                return m
            xe[:m].copy_(x_pin[r0:r1], non_blocking=True)
            if fused:
                for c0 in range(0, m, phi_ij_h.shape[0]):
                    c1 = min(m, c0 + phi_ij_h.shape[0])
                    pf, pij = ex.shap_and_interactions_device(xe[c0:c1], stream=stream)
                    phi_ij_h[:c1 - c0].copy_(pij, non_blocking=True)
                    phi_h[c0:c1].copy_(pf, non_blocking=True)
                return m
            if run.do_shap:
                ex.shap_device(xe[:m], out=run.phi[:m], stream=stream)
                phi_h[:m].copy_(run.phi[:m], non_blocking=True)
            if run.do_int:
                for c0, c1, chunk in ex.iter_interactions(xe[:m], phi_ij_h.shape[0], stream=stream, n_buffers=1):
                    phi_ij_h[:c1 - c0].copy_(chunk, non_blocking=True)
            return m

        # cold: the first call of a fresh model = preprocessing + one e2e step
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        m0 = e2e_step(0)
        b.record(stream)
        torch.cuda.synchronize()
        first_ms = a.elapsed_time(b)
        e2e_step(1)
        torch.cuda.synchronize()
        barrier(world)
        te, tr = [], []
        reps = max(2, min(args.steps // 2, 5))
        for i in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            tr.append(e2e_step(i))
            b.record(stream)
            torch.cuda.synchronize()
            te.append(a.elapsed_time(b))
        ms_e2e = max_over_ranks(float(np.mean(te)), world)
        rows_e2e = float(np.mean(tr))
        h2d = int(rows_e2e * M * run.esz)
        d2h = int(rows_e2e * ((G * (M + 1) * run.esz if run.do_shap else 0) + (run.ij_row_bytes if run.do_int else 0)))
        e2e = {"value": world * rows_e2e / (ms_e2e / 1000.0), "unit": "rows/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e, "steps": reps,
               "api": (f"TreeShapExplainer.explain_host_pipelined (pinned host X -> {args.e2e_chunks} chunks on "
                       "3 streams, H2D / kernel / D2H overlapped -> pinned host outputs)" if pipelined else
                       ("TreeShapExplainer.shap_and_interactions_device" if fused else
                        "TreeShapExplainer.shap_device/interactions_device") +
                       " with pinned host X and outputs (H2D + D2H)")}
        cold_s = pre_ms / 1000.0 + first_ms / 1000.0
        e2e_cold = {"value": world * m0 / cold_s, "unit": "rows/s", "rows": m0, "seconds": cold_s,
                    "preprocess_s": pre_ms / 1000.0, "first_call_s": first_ms / 1000.0,
                    "breakdown_s": {k: round(v, 4) for k, v in timings.items()},
                    "note": "fresh model: extract + pack + plan + blob write + H2D (+ broadcast) + one e2e step "
                            "(SURVEY §8(d) end to end)"}

    # --- ablation: the paper-lineage warp-bin kernels on a slice of the rows
    ablation = None
    if not args.no_ablation and rank == 0 and world == 1:
        na = min(run.rows_per_step, args.ablation_rows)
        xa = run.xd[:na]
        res = {"rows": na, "layout": "warp_bins (paper lineage: lane per path element, shuffles, swap-to-end)"}

        def timed1(fn, x, target_s=4.0):
            """rows/s of fn on a prefix of x sized for ~target_s of device time
            (a 256-row probe first: the paper-lineage kernel is ~50x slower)."""
            def once(xx):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(run.stream)
                fn(xx)
                b.record(run.stream)
                torch.cuda.synchronize()
                return a.elapsed_time(b) / 1000.0
            probe = x[:min(256, x.shape[0])]
            fn(probe)
            torch.cuda.synchronize()
            rate = probe.shape[0] / max(once(probe), 1e-6)
            m = int(min(x.shape[0], max(probe.shape[0], rate * target_s)))
            xx = x[:m]
            fn(xx)
            torch.cuda.synchronize()
            res["timed_rows"] = m
            return m / once(xx)

        packs = ["bfd", "ffd", "nf", "none"] if args.pack_ablation else [args.pack]
        for pk in packs:
            exb = TreeShapExplainer(ens, dtype=args.dtype, pack=pk, layout="warp_bins", device=dev,
                                    interactions=run.do_int and pk == args.pack)
            bv = exb.bins.view()
            ent = {"bins": int(bv["n_bins"]), "utilisation": bv["utilisation"]}
            if run.do_shap:
                ent["shap_rows_per_s"] = timed1(exb.shap_device, xa)
            if run.do_int and pk == args.pack:
                ni = max(1, min(na, run.ij_chunk, 8192))
                ent["interactions_rows_per_s"] = timed1(exb.interactions_device, xa[:ni])
                ent["interaction_rows"] = ni
            if pk == args.pack:
                res.update(ent)
            if args.pack_ablation:
                res.setdefault("packers", {})[pk] = ent
            del exb
        ablation = res

    peaks = measured_peaks()
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    f_max = (clocks["sm_max_mhz"] or peaks.get("sm_max_mhz", 1965.0)) * 1e6
    f_med = (clocks["sm_mhz"] or f_max / 1e6) * 1e6
    fp32_peak = sm_count * FP32_LANES_PER_SM * 2 * f_max / 1e12  # TFLOP/s
    if args.dtype == "f64":
        fp32_peak /= 2.0  # B200: FP64 at half the FP32 rate
    fpr, ppr = run.flops_per_row()
    roof = roofline(fpr, ppr, rows_step, ms_step, fp32_peak, f_med / f_max)
    roof["kernel"] = {"shap": "gts_shap", "interactions": "gts_shap_interactions",
                      "both": "gts_shap_and_interactions" if fused else "gts_shap + gts_shap_interactions"}[mode] + \
        f" ({args.layout} kernel + init fill, CUDA events on the launch stream)"
    roof["ms_median"], roof["ms_min"] = ms_med, ms_min
    tr = _traffic_entry(args.workload, args.layout, mode, args.dtype)
    if tr:
        rows_prof = tr.get("rows_per_launch")
        scale = (rows_step / rows_prof) if rows_prof else 1.0
        roof["traffic"] = tr.get("dram_bytes_per_launch") * scale
        roof["traffic_source"] = tr.get("source") + (f" (captured at {rows_prof} rows, scaled to {rows_step})"
                                                     if rows_prof and rows_prof != rows_step else "")
        if tr.get("executed_fp32_flops_per_row"):
            roof["ncu_executed_fp32_flops_per_row"] = tr["executed_fp32_flops_per_row"]
            roof["ncu_executed_over_nodal"] = tr["executed_fp32_flops_per_row"] / fpr
    roof["algorithmic_bytes_per_row"] = (M * run.esz + (G * (M + 1) * run.esz if run.do_shap else 0) +
                                         (run.ij_row_bytes if run.do_int else 0) + info_main.bytes / rows_step)

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_oracle_rates(w, ens, mode, args.cpu_seconds)

    extras = None
    if world == 1 and rank == 0 and args.extras != "none":
        spec = ("cal_housing-med:both:1048576,adult-large:both:65536,covtype-large:interactions:4096,"
                "fashion_mnist-med:shap:65536,fashion_mnist-med:interactions:1024" if args.extras == "auto"
                else args.extras)
        extras = {}
        for item in spec.split(","):
            name, xmode, xrows = item.split(":")
            extras[f"{name}:{xmode}"] = run_extra(args, name, xmode, int(xrows), dev, flush, fp32_peak, f_med / f_max)

    launches = run.launches_per_step()
    if rank != 0:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    total_rows = world * rows_step
    line = {
        "metric": METRIC,
        "value": total_rows / (ms_step / 1000.0),
        "unit": "rows/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "ms_per_step_median": ms_med,
        "ms_per_step_min": ms_min,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": args.dtype,
        "data": "synthetic",
        "config": {"workload": args.workload, "mode": mode, "rows_per_gpu": n, "rows_per_step": rows_step,
                   "global_rows_per_step": total_rows, "windows": len(run.windows),
                   "steps_note": "each step explains the next rows_per_step-row window of the resident "
                                 "rows_per_gpu-row dataset (windows rotate)",
                   "trees": w.n_trees, "max_depth": w.max_depth, "features": M, "groups": G,
                   "paths": int(info_main.n_paths), "path_elems": int(info_main.n_elems), "layout": args.layout,
                   "pack": args.pack, "x_layout": args.x_layout, "max_slots": int(info_main.max_slots),
                   "blob_bytes": int(info_main.bytes),
                   "bins": int(bins_view["n_bins"]) if bins_view else None,
                   "bin_utilisation": round(float(bins_view["utilisation"]), 6) if bins_view else None,
                   "phi_ij_chunk_rows": run.ij_chunk if run.do_int else None,
                   "l2": "flushed between timed steps (512 MiB memset outside the events)",
                   "parallelism": f"dp{world}: rows sharded, path table replicated by one NCCL broadcast"},
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "e2e_cold": e2e_cold,
        "gpu_launches": launches * args.steps,
        "gpu_launches_per_step": launches,
        "clocks": clocks,
        "preprocess_ms": pre_ms,
        "preprocess_breakdown_s": {k: round(v, 4) for k, v in timings.items()},
        "pack_seconds": bins_view["pack_seconds"] if bins_view else None,
        "broadcast_ms": bcast_ms,
        "extra": extras,
        "ablation_paper_kernels": ablation,
        "paper_v100_context": PAPER_V100.get(args.workload),
        "peak_source": f"FP32 {sm_count} SMs x {FP32_LANES_PER_SM} lanes x 2 x max SM clock (DESIGN.md §6); "
                       f"FFMA microbenchmark {FFMA_MEASURED_TFLOPS} TFLOP/s (profiles/r01c); "
                       f"HBM {peaks.get('hbm_gbs')} GB/s measured",
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_extra(args, name, mode, rows, dev, flush, peak, f_ratio):
    """A secondary workload at N=1 (same timing rules, 3 warm-up + 5 timed steps)."""
    import torch

    from paper_2010_13972_b200.explainer import TreeShapExplainer
    from synth.configs import WORKLOADS
    w = WORKLOADS[name]
    ens = w.ensemble()
    t0 = time.perf_counter()
    ex = TreeShapExplainer(ens, dtype=args.dtype, pack=args.pack, layout=args.layout, device=dev,
                           interactions=False, build_blobs=False)
    _ = ex.blob if mode == "shap" else ex.blob_int
    pre = time.perf_counter() - t0
    sub = argparse.Namespace(**vars(args))
    sub.x_layout = "row"
    run = Runner(sub, w, ex, mode, rows, rows, dev, 0)
    ms, rws = run.timed(5, 3, flush, 1)
    fpr, ppr = run.flops_per_row()
    r = roofline(fpr, ppr, rws[0], float(np.mean(ms)), peak, f_ratio)
    out = {"rows_per_step": rws[0], "rows_per_s": rws[0] / (float(np.mean(ms)) / 1000.0), "ms": float(np.mean(ms)),
           "ms_min": float(np.min(ms)), "frac_nodal": r["frac_nodal"], "frac_survey_8d": r["frac_survey_8d"],
           "achieved_tflops": r["achieved"], "preprocess_s": pre,
           "call": {"shap": "gts_shap", "interactions": "gts_shap_interactions",
                    "both": "gts_shap_and_interactions"}[mode], "paper_v100_context": PAPER_V100.get(name)}
    del run, ex
    torch.cuda.empty_cache()
    return out


def run_sweep(args):
    """Latency regime (Fig. 4): per row
    count, the device time of one SHAP call issued eagerly (init + main kernel
    launches through the C ABI) and replayed from a CUDA graph, beside the
    oracle (fp64, all host cores) on the same rows; prints one JSON line."""
    import torch

    import oracle
    from paper_2010_13972_b200.explainer import TreeShapExplainer
    from synth.configs import WORKLOADS

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    w = WORKLOADS[args.workload]
    ens = w.ensemble()
    ex = TreeShapExplainer(ens, dtype=args.dtype, pack=args.pack, layout=args.layout, device=dev,
                           interactions=False)
    stream = torch.cuda.current_stream(dev)
    points = []
    n_max = int(args.rows_per_gpu)
    counts = [c for c in (1, 4, 16, 64, 256, 1024, 4096, 16384, 65536, 262144, 1 << 20) if c <= n_max]
    x_all = w.x(max(counts), ens=ens if w.tie_frac > 0 else None)
    xd_all = torch.from_numpy(x_all if args.dtype == "f32" else x_all.astype(np.float64)).to(dev)
    for n in counts:
        xd = xd_all[:n]
        out = torch.empty((n, w.n_groups, w.n_features + 1), dtype=xd.dtype, device=dev)
        reps = 50 if n <= 4096 else (10 if n <= 65536 else 3)

        def timed(fn):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            ts = []
            for _ in range(reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                fn()
                b.record(stream)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b) * 1000.0)
            return float(np.median(ts))

        # eager: back-to-back calls so the host launch cost is part of the device timeline
        eager = timed(lambda: ex.shap_device(xd, out=out, stream=stream))
        g = ex.graphed(n)
        g.x.copy_(xd)
        graph = timed(g.replay)
        del g
        cpu_us = None
        if n <= 4096:
            xr = x_all[:n].astype(np.float64)
            t0 = time.perf_counter()
            r = 0
            while True:
                oracle.treeshap(ens, xr)
                r += 1
                if time.perf_counter() - t0 > 0.2 or r >= 20:
                    break
            cpu_us = (time.perf_counter() - t0) / r * 1e6
        points.append({"rows": n, "eager_us": eager, "graph_us": graph, "cpu_oracle_us": cpu_us,
                       "graph_rows_per_s": n / (graph * 1e-6)})
    cross = next((p["rows"] for p in points if p["cpu_oracle_us"] is not None and p["cpu_oracle_us"] > p["graph_us"]),
                 None)
    print(json.dumps({"sweep": "latency", "workload": args.workload, "dtype": args.dtype, "layout": args.layout,
                      "points": points, "gpu_faster_from_rows": cross,
                      "cpu_cores": oracle.num_threads(),
                      "note": "device time per SHAP call (CUDA events, median); cpu = fp64 oracle wall time"}),
          flush=True)


def main():
    args = parse()
    if args.latency_sweep:
        run_sweep(args)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

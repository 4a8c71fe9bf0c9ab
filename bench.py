"""Benchmark: exact path-wise TreeShap rows/s on B200 (SHAP + interaction
values), with roofline fraction, CPU-oracle baseline, clocks and an end-to-end
number through the public API.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cal_housing-med] [--rows-per-gpu 1048576] [--mode both|shap|interactions]

One "step" = one pass of the per-row hot path over this rank's batch of rows
producing the SHAP values + bias and the interaction values: in mode "both"
one gts_shap_and_interactions call (the interaction kernel also writes phi;
`--separate` times gts_shap + gts_shap_interactions instead, which the line
reports beside it as "both.separate_*", and "shap" / "interactions" time each
kernel alone), with the packed path table resident (extract -> pack -> blob runs once per model,
PAPER.md:528, and is reported as `preprocess_ms`).  Rows are sharded across
ranks (weak scaling); the blob is replicated by ONE NCCL broadcast.  Rank 0
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
    ap.add_argument("--workload", default="cal_housing-med")
    ap.add_argument("--rows-per-gpu", type=int, default=1 << 20)
    ap.add_argument("--mode", choices=["both", "shap", "interactions"], default="both")
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

def run_ours(args):
    import torch

    from paper_2010_13972_b200 import gts
    from paper_2010_13972_b200.explainer import Blob, TreeShapExplainer
    from synth.configs import WORKLOADS

    world, rank, local = dist_setup(args)
    dev = torch.device("cuda", local)
    w = WORKLOADS[args.workload]
    ens = w.ensemble()
    M, G = w.n_features, w.n_groups
    n = int(args.rows_per_gpu)
    do_shap = args.mode in ("both", "shap")
    do_int = args.mode in ("both", "interactions")

    # --- model preprocessing: rank 0 extracts + packs + writes the blob; one broadcast
    t0 = time.perf_counter()
    if rank == 0:
        ex = TreeShapExplainer(ens, dtype=args.dtype, pack=args.pack, layout=args.layout, device=dev,
                               interactions=do_int, max_slots=args.max_slots)
    else:
        ex = TreeShapExplainer(ens, dtype=args.dtype, pack=args.pack, layout=args.layout, device=dev,
                               interactions=do_int, build_blobs=False, max_slots=args.max_slots)
        ex.blob = Blob(None, torch.empty(0, dtype=torch.uint8, device=dev))
        ex.blob_int = Blob(None, torch.empty(0, dtype=torch.uint8, device=dev)) if do_int else None
    torch.cuda.synchronize()
    pre_ms = 1000 * (time.perf_counter() - t0)
    bcast_ms = 0.0
    if world > 1:
        # every rank knows whether the interaction kernel reuses the SHAP blob
        same = args.layout == "warp_bins" or M <= 16
        barrier(world)
        t1 = time.perf_counter()
        ex.blob.broadcast(0)
        if do_int:
            ex.blob_int = ex.blob if same else ex.blob_int.broadcast(0)
        torch.cuda.synchronize()
        bcast_ms = 1000 * (time.perf_counter() - t1)
    info_s, info_i = ex.blob.info, (ex.blob_int.info if do_int else None)
    bins_view = ex.bins.view()

    # --- this rank's rows (counter-keyed generator: no scatter)
    x_host = w.x(n, row0=rank * n, ens=ens if w.tie_frac > 0 else None)
    xh = x_host if args.dtype == "f32" else x_host.astype(np.float64)
    if args.x_layout == "feature":  # [n][M] view of a feature-major [M][n] buffer
        xt = torch.from_numpy(np.ascontiguousarray(xh.T)).t()
    else:
        xt = torch.from_numpy(xh)
    xd = xt.to(dev)
    x_rs, x_cs = TreeShapExplainer._strides(xd)
    tdt = torch.float32 if args.dtype == "f32" else torch.float64
    phi = torch.empty((n, G, M + 1), dtype=tdt, device=dev) if do_shap else None
    # wide models (fashion_mnist: 24.6 MB of phi_ij per row) stream the rows in
    # chunks through one reused buffer; otherwise one call
    ij_row_bytes = G * (M + 1) ** 2 * (4 if args.dtype == "f32" else 8)
    ij_chunk = n if not do_int else max(1, min(n, (args.phi_ij_budget_gb << 30) // ij_row_bytes))
    phi_ij = torch.empty((ij_chunk, G, M + 1, M + 1), dtype=tdt, device=dev) if do_int else None
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    fused = args.mode == "both" and not args.separate

    def fused_step(evs=None):
        if evs: evs[4].record(stream)
        for r0 in range(0, n, ij_chunk):
            xr = xd[r0:r0 + ij_chunk]
            gts.gts_shap_and_interactions(info_i, ex.blob_int.ptr, xr.data_ptr(), xr.shape[0], x_rs, x_cs,
                                          phi[r0:r0 + ij_chunk].data_ptr(), phi_ij.data_ptr(), stream.cuda_stream)
        if evs: evs[5].record(stream)

    def step(evs=None):
        if do_shap:
            if evs: evs[0].record(stream)
            gts.gts_shap_strided(info_s, ex.blob.ptr, xd.data_ptr(), n, x_rs, x_cs, phi.data_ptr(),
                                 stream.cuda_stream)
            if evs: evs[1].record(stream)
        if do_int:
            if evs: evs[2].record(stream)
            for r0 in range(0, n, ij_chunk):
                xr = xd[r0:r0 + ij_chunk]
                gts.gts_shap_interactions_strided(info_i, ex.blob_int.ptr, xr.data_ptr(), xr.shape[0], x_rs, x_cs,
                                                  phi_ij.data_ptr(), stream.cuda_stream)
            if evs: evs[3].record(stream)

    for _ in range(args.warmup):
        step()
        if fused:
            fused_step()
    torch.cuda.synchronize()
    gpu_uuid = str(torch.cuda.get_device_properties(dev).uuid)
    gpu_id = gpu_uuid if gpu_uuid.startswith("GPU-") else "GPU-" + gpu_uuid
    t_step, t_shap, t_int, t_sep = [], [], [], []
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(gpu_id) as clk:
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
            step(evs)
            if fused:
                flush.zero_()
                fused_step(evs)
            torch.cuda.synchronize()
            ts = evs[0].elapsed_time(evs[1]) if do_shap else 0.0
            ti = evs[2].elapsed_time(evs[3]) if do_int else 0.0
            t_shap.append(ts)
            t_int.append(ti)
            t_sep.append(ts + ti)
            t_step.append(evs[4].elapsed_time(evs[5]) if fused else ts + ti)
    torch.cuda.synchronize()
    barrier(world)
    ms_step = max_over_ranks(float(np.mean(t_step)), world)
    ms_sep = max_over_ranks(float(np.mean(t_sep)), world)
    ms_shap = max_over_ranks(float(np.mean(t_shap)), world)
    ms_int = max_over_ranks(float(np.mean(t_int)), world)
    clocks = clk.summary()

    # --- end to end through the public API: pinned host X -> device -> host phi
    e2e = None
    if not args.no_e2e:
        x_pin = xt.pin_memory()
        phi_h = torch.empty(phi.shape, dtype=tdt, pin_memory=True) if do_shap else None
        e2e_chunk = max(1, min(ij_chunk, (4 << 30) // ij_row_bytes))  # pinned host staging <= 4 GiB
        phi_ij_h = torch.empty((e2e_chunk,) + tuple(phi_ij.shape[1:]), dtype=tdt, pin_memory=True) if do_int else None
        xe = torch.empty_like(xd)

        pipelined = not args.e2e_serial and ij_chunk == n and args.x_layout == "row"
        if pipelined:
            phi_ij_h = torch.empty(tuple(phi_ij.shape), dtype=tdt, pin_memory=True) if do_int else None
            del phi_ij  # the pipelined call has its own device slots
            torch.cuda.empty_cache()

        def e2e_step():
            if pipelined:
                ex.explain_host_pipelined(x_pin, phi_h, phi_ij_h, chunk_rows=max(1, -(-n // args.e2e_chunks)))
                return
            xe.copy_(x_pin, non_blocking=True)
            if fused:
                for r0 in range(0, n, e2e_chunk):
                    r1 = min(n, r0 + e2e_chunk)
                    ex.shap_and_interactions_device(xe[r0:r1], out_phi=phi[r0:r1], out_phi_ij=phi_ij[: r1 - r0],
                                                    stream=stream)
                    phi_ij_h[: r1 - r0].copy_(phi_ij[: r1 - r0], non_blocking=True)
                phi_h.copy_(phi, non_blocking=True)
                return
            if do_shap:
                ex.shap_device(xe, out=phi, stream=stream)
                phi_h.copy_(phi, non_blocking=True)
            if do_int:
                for r0, r1, chunk in ex.iter_interactions(xe, e2e_chunk, stream=stream, n_buffers=1):
                    phi_ij_h[: r1 - r0].copy_(chunk, non_blocking=True)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        barrier(world)
        te = []
        for _ in range(max(2, args.steps // 2)):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            e2e_step()
            b.record(stream)
            torch.cuda.synchronize()
            te.append(a.elapsed_time(b))
        ms_e2e = max_over_ranks(float(np.mean(te)), world)
        h2d = xt.numel() * xt.element_size()
        d2h = (phi.numel() * phi.element_size() if do_shap else 0) + (n * ij_row_bytes if do_int else 0)
        e2e = {"value": world * n / (ms_e2e / 1000.0), "unit": "rows/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": ms_e2e,
               "api": (f"TreeShapExplainer.explain_host_pipelined (pinned host X -> {args.e2e_chunks} chunks on "
                       "3 streams, H2D / kernel / D2H overlapped -> pinned host phi and phi_ij)" if pipelined else
                       ("TreeShapExplainer.shap_and_interactions_device" if fused else
                        "TreeShapExplainer.shap_device/interactions_device") +
                       " with pinned host X and phi (H2D + D2H)")}

    # --- ablation: the paper-lineage warp-bin kernels on a slice of the rows
    ablation = None
    if not args.no_ablation and rank == 0:
        # the paper-lineage warp-bin kernels on a slice of the rows; with
        # --pack-ablation every packer's bins (utilisation ->
        # kernel time), SHAP only
        na = min(n, args.ablation_rows)
        xa = xd[:na]
        res = {"rows": na, "layout": "warp_bins (paper lineage: lane per path element, shuffles, swap-to-end)"}

        def timed(fn, x):
            fn(x)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn(x)
            b.record(stream)
            torch.cuda.synchronize()
            return x.shape[0] / (a.elapsed_time(b) / 1000.0)

        packs = ["bfd", "ffd", "nf", "none"] if args.pack_ablation else [args.pack]
        for pk in packs:
            exb = TreeShapExplainer(ens, dtype=args.dtype, pack=pk, layout="warp_bins", device=dev,
                                    interactions=do_int and pk == args.pack)
            bv = exb.bins.view()
            ent = {"bins": int(bv["n_bins"]), "utilisation": bv["utilisation"]}
            if do_shap:
                ent["shap_rows_per_s"] = timed(exb.shap_device, xa)
            if do_int and pk == args.pack:
                ni = max(1, min(na, ij_chunk, 8192))
                ent["interactions_rows_per_s"] = timed(exb.interactions_device, xa[:ni])
                ent["interaction_rows"] = ni
            if pk == args.pack:
                res.update(ent)
            if args.pack_ablation:
                res.setdefault("packers", {})[pk] = ent
            del exb
        ablation = res

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_oracle_rates(w, ens, args.mode, args.cpu_seconds)

    if rank != 0:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return

    peaks = measured_peaks()
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    f_max = (clocks["sm_max_mhz"] or peaks.get("sm_max_mhz", 1965.0)) * 1e6
    f_med = (clocks["sm_mhz"] or f_max / 1e6) * 1e6
    fp32_peak = sm_count * FP32_LANES_PER_SM * 2 * f_max / 1e12  # TFLOP/s
    if args.dtype == "f64":
        fp32_peak /= 2.0  # B200: FP64 at half the FP32 rate
    total_rows = world * n

    def roof(flops_per_row, paper_flops_per_row, ms):
        if ms <= 0:
            return None
        ach = flops_per_row * n / (ms / 1000.0) / 1e12
        return {"bound": "alu", "achieved": ach, "peak": fp32_peak, "unit": "TFLOP/s", "frac": ach / fp32_peak,
                "frac_at_median_clock": ach / (fp32_peak * f_med / f_max), "traffic": None,
                "flops_per_row": flops_per_row,
                "paper_recurrence_equiv_tflops": paper_flops_per_row * n / (ms / 1000.0) / 1e12}

    r_shap = roof(info_s.shap_flops_per_row, info_s.paper_shap_flops_per_row, ms_shap) if do_shap else None
    r_int = roof(info_i.inter_flops_per_row, info_i.paper_inter_flops_per_row, ms_int) if do_int else None
    dominant = "interactions" if (do_int and ms_int >= ms_shap) else "shap"
    if fused:
        # the step is the fused call: the interaction kernel's work, phi read off its diagonal
        r_both = roof(info_i.inter_flops_per_row, info_i.paper_inter_flops_per_row, ms_step)
        roofline = dict(r_both)
        roofline["kernel"] = (f"gts_shap_and_interactions ({args.layout} interaction kernel writing phi and phi_ij "
                              "+ init fills, CUDA events on the launch stream)")
    else:
        roofline = dict((r_int if dominant == "interactions" else r_shap) or {})
        roofline["kernel"] = ("gts_shap_interactions" if dominant == "interactions" else "gts_shap") + \
            f" ({args.layout} kernel + init fill, CUDA events on the launch stream)"
    traffic_file = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(traffic_file):
        try:
            tr = json.load(open(traffic_file)).get(
                f"{args.workload}/{args.layout}/{'both' if fused else dominant}/{args.dtype}")
            if tr:
                roofline["traffic"] = tr.get("dram_bytes_per_launch")
                roofline["traffic_source"] = tr.get("source")
        except Exception:
            pass
    launches_sep = (gts.gts_launches_per_call(info_s, False) if do_shap else 0) + (
        gts.gts_launches_per_call(info_i, True) * -(-n // ij_chunk) if do_int else 0)
    launches = gts.gts_launches_per_call(info_i, 2) * -(-n // ij_chunk) if fused else launches_sep
    line = {
        "metric": METRIC,
        "value": total_rows / (ms_step / 1000.0),
        "unit": "rows/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": args.dtype,
        "data": "synthetic",
        "config": {"workload": args.workload, "mode": args.mode, "rows_per_gpu": n, "global_rows": total_rows,
                   "trees": w.n_trees, "max_depth": w.max_depth, "features": M, "groups": G,
                   "paths": int(info_s.n_paths), "path_elems": int(info_s.n_elems), "layout": args.layout,
                   "pack": args.pack, "x_layout": args.x_layout, "max_slots": int(info_s.max_slots), "bins": int(bins_view["n_bins"]),
                   "bin_utilisation": round(float(bins_view["utilisation"]), 6),
                   "phi_ij_chunk_rows": ij_chunk if do_int else None,
                   "l2": "flushed between timed steps (512 MiB memset outside the events); phi_ij > L2",
                   "parallelism": f"dp{world}: rows sharded, path table replicated by one NCCL broadcast"},
        "shap": {"rows_per_s": total_rows / (ms_shap / 1000.0), "ms": ms_shap, "roofline": r_shap} if do_shap else None,
        "interactions": {"rows_per_s": total_rows / (ms_int / 1000.0), "ms": ms_int, "roofline": r_int}
        if do_int else None,
        "both": ({"rows_per_s": total_rows / (ms_step / 1000.0), "ms": ms_step,
                  "call": "gts_shap_and_interactions (one pass: phi and phi_ij)",
                  "separate_rows_per_s": total_rows / (ms_sep / 1000.0), "separate_ms": ms_sep,
                  "separate_launches_per_step": launches_sep} if fused else None),
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches * args.steps,
        "gpu_launches_per_step": launches,
        "clocks": clocks,
        "preprocess_ms": pre_ms,
        "pack_seconds": bins_view["pack_seconds"],
        "broadcast_ms": bcast_ms,
        "ablation_paper_kernels": ablation,
        "paper_v100_context": PAPER_V100.get(args.workload),
        "peak_source": f"FP32 {sm_count} SMs x {FP32_LANES_PER_SM} lanes x 2 x max SM clock (DESIGN.md §6); "
                       f"HBM {peaks.get('hbm_gbs')} GB/s measured",
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


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

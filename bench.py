#!/usr/bin/env python
"""bench.py -- GSCache fit+query step throughput on B200 (BASELINE.json metric).

A step is one frame of the paper's per-frame loop (sec.3.1): the full-frame cache
lookup (the "ST" analogue, Table 2) and one optimisation step on the frame's noisy
renderer samples (the "OT" analogue): ingest + binning, fused fwd + HDR loss + bwd, AdamW,
culling rebuild -- one gc_fit_query call (lookups read the pre-step cache and overlap the
fit half on an internal stream; --separate times gc_query + gc_fit instead).  Workload: BASELINE configs[2] (4 levels 65,536/16,384/4,096/1,024
Gaussians, one 1920x1080 frame = 2,073,600 samples per step), synthetic (workload.py).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

N > 1 runs under torchrun: one process per GPU, every rank fits its own frame (weak scaling)
and one NCCL all-reduce of the level gradients per step keeps the replicas identical.
Rank 0 prints ONE JSON line.
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

import workload  # noqa: E402

FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12     # 74.45 TFLOP/s (DESIGN.md derivation)
FLOPS_PER_PAIR = 67.0                                  # fwd 30 + bwd 37 per pair
FLOPS_PER_SAMPLE = 20.0                                # loss + dL/dy per fitted sample
FLOPS_PER_QPAIR = 30.0


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class Clocks:
    """nvidia-smi sampler running during the timed region (the recipe's clocks line)."""

    def __init__(self, index=0):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 4 + k and r[4 + k].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    """The fp64 CPU oracle as it stands, on the host cores, bounded sample per step."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle
    cfg = args.config
    c = workload.CONFIGS[cfg]
    pos, alb = workload.init_cloud(cfg)
    counts = c["counts"]
    # untimed setup: the oracle's create with Eq. 2 scales per level; the 3-NN means come from
    # scipy's k-d tree (the oracle's O(N^2) brute force would take minutes at 65k points),
    # then oracle.eq2_from_dbar applies Eq. 2 itself.
    from scipy.spatial import cKDTree
    P = oracle.create(counts, pos.astype(np.float64), alb.astype(np.float64),
                      np.zeros((counts[0], 3)), seed=cfg)
    goff = np.concatenate([[0], np.cumsum(counts)])
    for l in range(len(counts)):
        pts = P[goff[l]:goff[l + 1], 0:3]
        d, _ = cKDTree(pts).query(pts, k=4)
        s_ = oracle.eq2_from_dbar(d[:, 1:].mean(1), oracle.diag(pts))
        P[goff[l]:goff[l + 1], 10:13] = np.log(s_)[:, None]
    grids = auto_grids(P, counts)
    oc = oracle.OracleCache(counts, P, grids=grids)
    n = args.ref_samples
    times = []
    for s in range(args.warmup + args.steps):
        x, ln, rgb = workload.fit_batch(cfg, frame=s % 4, S=n)
        xq, lq = workload.query_batch(cfg, frame=s % 4, S=n)
        t0 = time.perf_counter()
        oc.query(xq.astype(np.float64), lq)
        r = oc.fit(x.astype(np.float64), ln, rgb.astype(np.float64))
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append((dt, int(r["count"].sum())))
    t = sum(d for d, _ in times) / len(times)
    nv = sum(k for _, k in times) / len(times)
    val = nv / t
    line = {"impl": "reference", "metric": metric_name(cfg), "value": val,
            "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": c["name"], "levels": len(counts), "counts": counts,
                       "S_per_step": n, "note": "oracle step on a bounded sample of the frame"},
            "cpu_baseline": {"value": val, "unit": "samples/s", "cores": 1, "kind": "oracle",
                             "sample": f"{n} fit samples + {n} queries per step of {c['name']}"},
            "e2e": {"value": val, "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def auto_grids(P, counts, tau=3.0):
    """Grid for the oracle-only reference arm (the oracle reads any grid; C8)."""
    goff = np.concatenate([[0], np.cumsum(counts)])
    out = []
    for l in range(len(counts)):
        Pl = P[goff[l]:goff[l + 1]]
        lo, hi = Pl[:, 0:3].min(0), Pl[:, 0:3].max(0)
        d = np.linalg.norm(hi - lo)
        lo, hi = lo - 0.05 * d - 1e-6, hi + 0.05 * d + 1e-6
        edge = 2 * tau * np.exp(Pl[:, 10:13]).mean()
        dims = np.clip(np.ceil((hi - lo) / edge), 1, 512).astype(np.int32)
        out.append((lo, dims / (hi - lo), dims))
    return out


def metric_name(cfg):
    return "cache samples fitted/s (fit+query step, fwd+bwd+AdamW)"


# ------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2507_19718_b200 as gsc

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = args.config
    c = workload.CONFIGS[cfg]
    counts = c["counts"]
    S = c["S"]
    pos, alb = workload.init_cloud(cfg)
    cache = gsc.GSCache(counts, torch.from_numpy(pos).to(dev), torch.from_numpy(alb).to(dev),
                        seed=cfg, device=local, hparams=dict(cell_edge_scale=args.cell_scale))
    if world > 1:
        uid = [gsc.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        cache.set_comm(uid[0], rank, world)
    R = 4                                   # rotating frames: inputs of step k last used 4 steps ago
    frames = []
    for f in range(R):
        x, ln, rgb = workload.fit_batch(cfg, frame=rank * R + f, morton=args.morton)
        xq, lq = workload.query_batch(cfg, frame=rank * R + f, morton=args.morton)
        frames.append(tuple(torch.from_numpy(a).to(dev) for a in (x, ln, rgb, xq, lq)))
    in_bytes = sum(t.numel() * t.element_size() for t in frames[0])
    outq = torch.empty((S, 3), dtype=torch.float32, device=dev)
    cache.reserve(S, S)
    stream = torch.cuda.Stream(device=dev)
    if not args.no_defer:       # each frame's optimizer step overlaps the next frame's ingest
        cache.set_deferred_step(True)

    def frame_call(x, ln, rgb, xq, lq, out, s_, separate=args.separate):
        if separate:                        # two calls, serialised on one stream
            cache.query(xq, lq, out=out, stream=s_)
            return cache.fit(x, ln, rgb, stream=s_)
        # one call: the lookups overlap the fit samples' ingest and fwd/bwd (internal stream)
        return cache.fit_query(x, ln, rgb, xq, lq, out=out, stream=s_)[1]

    def step(f, s_):
        return frame_call(*frames[f], outq, s_)

    # warm-up (eager), then capture one CUDA graph per rotating frame
    with torch.cuda.stream(stream):
        for w in range(max(args.warmup, 1)):
            step(w % R, stream)
    stream.synchronize()
    graphs = []
    if not args.no_graph:
        for f in range(R):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                step(f, stream)
            graphs.append(g)
        with torch.cuda.stream(stream):
            for w in range(args.warmup):
                graphs[w % R].replay()
    stream.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # ---- timed region (device time, CUDA events on the launching stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier()
        e0.record(stream)
        with torch.cuda.stream(stream):
            for k in range(args.steps):
                if graphs:
                    graphs[k % R].replay()
                else:
                    step(k % R, stream)
            cache.flush(stream)        # the last frame's deferred step is inside the timed region
        e1.record(stream)
        barrier()
        ms_total = e0.elapsed_time(e1)
        ms = torch.tensor([ms_total / args.steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        ms_step = float(ms.item())
        if args.clock_window > 0:     # keep the GPU busy long enough for nvidia-smi samples;
            # the same number of frames on every rank (each frame holds an NCCL all-reduce)
            rounds = max(1, int(args.clock_window * 1e3 / (ms_step * 20)))
            with torch.cuda.stream(stream):
                for _ in range(rounds):
                    for k in range(20):
                        (graphs[k % R].replay() if graphs else step(k % R, stream))
                    stream.synchronize()
    st = cache._stats
    torch.cuda.synchronize(dev)
    n_valid = int(st.n_valid)           # last step's valid samples (global under DP)
    n_valid_local = n_valid // world if world > 1 else n_valid
    value = n_valid_local * world / (ms_step * 1e-3)

    # ---- per-kernel device time of the same steps, eager with events per kernel, the two
    # halves serialised (gc_query + gc_fit) so that no kernel's time includes an overlap
    cache.set_deferred_step(False)
    cache.flush(stream)
    cache.profile_enable(True)
    cache.profile_read(reset=True)
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e2.record(stream)
    with torch.cuda.stream(stream):
        for k in range(args.steps):
            frame_call(*frames[k % R], outq, stream, separate=True)
    e3.record(stream)
    torch.cuda.synchronize(dev)
    prof = cache.profile_read(reset=True)
    cache.profile_enable(False)
    cache.set_deferred_step(not args.no_defer)
    ms_eager = e2.elapsed_time(e3) / args.steps
    launches_per_step = sum(v[1] for v in prof.values()) / args.steps
    kernel_ms = {k: v[0] / max(v[1], 1) for k, v in prof.items()}
    share = {k: v[0] / args.steps / ms_eager for k, v in prof.items()}
    top = max(prof, key=lambda k: prof[k][0])
    n_pairs, n_cand = int(st.n_pairs), int(st.n_candidates)
    pk, pk_kind = peaks()
    traffic, traffic_src = None, None
    try:   # per-launch DRAM bytes of the dominant kernel from the committed ncu launch list
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        traffic = next((v for k, v in tj["bytes_per_launch"].items() if k.endswith("k_" + top) or
                        k.endswith("k_" + top + "<0>")), None)
        traffic_src = "profiles/traffic.json: " + tj["source"]
    except Exception:
        pass
    issue = None
    try:   # the kernel's issue rate from the committed ncu capture (its real limiter)
        with open(os.path.join(ROOT, "profiles", "issue.json")) as f:
            ij = json.load(f)
        m = ij["kernels"].get("k_" + top)
        if m:
            issue = {"ipc": m["ipc"], "peak_ipc": 4.0, "frac": m["ipc"] / 4.0,
                     "fma_pipe_pct": m["fma_pipe_pct"], "xu_pipe_pct": m["xu_pipe_pct"],
                     "source": "profiles/issue.json: " + ij["source"]}
    except Exception:
        pass
    if top == "fwdbwd":
        flops = (n_pairs / world) * FLOPS_PER_PAIR + n_valid_local * FLOPS_PER_SAMPLE
        achieved = flops / (kernel_ms[top] * 1e-3) / 1e12
        roof = {"bound": "alu", "achieved": achieved, "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP32_PEAK_TFLOPS, "traffic": traffic, "kernel": top,
                "traffic_source": traffic_src,
                "peak_source": "derived: 148 SM x 128 FP32 lanes x 2 x 1.965 GHz (B200_PROFILING.md counts/clock)",
                "algorithmic": f"{FLOPS_PER_PAIR:.0f} flop/contributing pair + {FLOPS_PER_SAMPLE:.0f}/sample",
                "issue_bound": issue}
    else:
        roof = {"bound": "hbm", "achieved": None, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": None, "traffic": None, "kernel": top}

    # ---- end to end through the public API with pinned HOST buffers
    hx = [tuple(t.cpu().pin_memory() for t in fr) for fr in frames]
    hout = torch.empty((S, 3), dtype=torch.float32).pin_memory()
    e4, e5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        for w in range(2):
            frame_call(*hx[w % R], hout, stream)
    barrier()
    e4.record(stream)
    with torch.cuda.stream(stream):
        for k in range(args.steps):
            frame_call(*hx[k % R], hout, stream)
        cache.flush(stream)
    e5.record(stream)
    barrier()
    ms_e2e = torch.tensor([e4.elapsed_time(e5) / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_e2e, op=dist.ReduceOp.MAX)
    ms_e2e = float(ms_e2e.item())
    e2e_val = n_valid_local * world / (ms_e2e * 1e-3)

    # ---- CPU oracle baseline (rank 0, N = 1 only), bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cache, cfg, args.cpu_samples or S)

    if rank == 0:
        line = {
            "metric": metric_name(cfg), "value": value, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": c["name"], "levels": len(counts), "counts": counts,
                       "S_fit_per_gpu": S, "S_query_per_gpu": S, "parallelism": f"dp{world}",
                       "l2": f"{R} rotating device-resident frames ({R * in_bytes / 1e6:.0f} MB) > 126 MB L2",
                       "cuda_graph": not args.no_graph,
                       "frame_call": "gc_query + gc_fit" if args.separate else "gc_fit_query",
                       "deferred_step": not args.no_defer,
                       "sample_order": "morton" if args.morton else "random"},
            "queries_per_s": S * world / (ms_step * 1e-3),
            "pairs_per_sample": n_pairs / max(n_valid, 1),
            "candidates_per_sample": n_cand / max(n_valid, 1),
            "roofline": roof,
            "kernel_ms": kernel_ms, "kernel_share_eager": share, "ms_per_step_eager": ms_eager,
            "e2e": {"value": e2e_val, "unit": "samples/s",
                    "h2d_bytes_per_step": int(in_bytes),
                    "d2h_bytes_per_step": int(S * 12 + 256)},
            "gpu_launches": int(round(launches_per_step * args.steps)),
            "clocks": clk.summary(), "peaks": pk_kind,
        }
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def cpu_baseline(cache, cfg, n):
    """The fp64 oracle on this box's host cores (1 thread): one fit + query step on a bounded
    sample of the same frame, starting from the same parameters and culling grids."""
    import oracle
    P = np.concatenate([cache.params_rows(l) for l in range(cache.L)]).astype(np.float64)
    oc = oracle.OracleCache(cache.counts, P, grids=cache.grids())
    x, ln, rgb = workload.fit_batch(cfg, frame=0, S=n)
    xq, lq = workload.query_batch(cfg, frame=0, S=n)
    t0 = time.perf_counter()
    oc.query(xq.astype(np.float64), lq)
    r = oc.fit(x.astype(np.float64), ln, rgb.astype(np.float64))
    dt = time.perf_counter() - t0
    return {"value": int(r["count"].sum()) / dt, "unit": "samples/s", "cores": 1, "kind": "oracle",
            "sample": f"{n} fit samples + {n} queries of {workload.CONFIGS[cfg]['name']} frame 0 "
                      f"(culled fp64 oracle, single thread, {dt:.1f} s)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--morton", action="store_true",
                    help="samples in Morton order (a screen-coherent renderer) instead of random order")
    ap.add_argument("--no-defer", action="store_true",
                    help="complete each frame's optimizer step inside its own call (no deferral)")
    ap.add_argument("--separate", action="store_true",
                    help="time gc_query + gc_fit instead of the gc_fit_query frame call")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-samples", type=int, default=0,
                    help="samples (and lookups) of the oracle baseline; 0 = the whole frame")
    ap.add_argument("--ref-samples", type=int, default=100_000)
    ap.add_argument("--clock-window", type=float, default=2.0)
    ap.add_argument("--cell-scale", type=float, default=1.0, help="culling-grid cell edge multiplier")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""bench.py -- GSCache fit+query step throughput on B200 (BASELINE.json metric).

A step is one frame of the paper's per-frame loop (sec.3.1): the full-frame cache
lookup (the "ST" analogue, Table 2) and one optimisation step on the frame's noisy
renderer samples (the "OT" analogue): ingest + binning, fused fwd + HDR loss + bwd, AdamW,
culling rebuild -- one gc_fit_query call (lookups read the pre-step cache and overlap the
fit half on an internal stream; --separate times gc_query + gc_fit instead).  Workload: BASELINE configs[2] (4 levels 65,536/16,384/4,096/1,024
Gaussians, one 1920x1080 frame = 2,073,600 samples per step), synthetic (workload.py).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]
                  [--scaling weak|strong] [--parallelism dp|level]

--gpus N > 1 runs one process per GPU: launched by torchrun (the driver), or, when WORLD_SIZE is
unset, bench.py re-executes itself under `python -m torch.distributed.run`.  --scaling weak
(default): every rank fits its own full frame of the config; strong: the config's frame is
split over the ranks (S/N samples and lookups each; cfg4's 16.8 M is the north star's case).
--parallelism dp (default): mode 0, one NCCL all-reduce of the level gradients per step keeps
the replicas identical; level: mode 1, samples and lookups are routed to the ranks owning
their level; oc: mode 2, spatial owner-computes with boundary-only exchanges (modes 1 and 2
are eager calls, not graph-capturable).  At N > 1 the other modes are timed too ("alt").  Rank 0 prints ONE JSON line.
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


def relaunch_under_torchrun(n):
    """--gpus N > 1 without a torchrun environment: re-execute this script as N ranks."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__),
           *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def cpu_info():
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except Exception:
        usable = os.cpu_count()
    return {"cpu_count": os.cpu_count(), "usable_cores": usable, "model": model}


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
def make_frames(cfg, rank, world, R, strong, morton, dev):
    """R rotating frames of device-resident inputs for this rank.  Weak scaling: the rank's
    own full frame of the config; strong: its 1/world slice of a global frame (each slice an
    independent seeded draw of the same distribution, S_global / world samples)."""
    import torch
    S = workload.CONFIGS[cfg]["S"]
    S_local = -(-S // world) if strong else S
    frames = []
    for f in range(R):
        fr = (f * 1000 + rank) if strong else (rank * R + f)
        x, ln, rgb = workload.fit_batch(cfg, frame=fr, S=S_local, morton=morton)
        xq, lq = workload.query_batch(cfg, frame=fr, S=S_local, morton=morton)
        frames.append(tuple(torch.from_numpy(a).to(dev) for a in (x, ln, rgb, xq, lq)))
    return frames, S_local


def level_weights(cfg, frames):
    """Mode-1 plan weights: each level's share of the frame's valid samples (the evaluator
    work) averaged with its share of the Gaussians (the optimizer work)."""
    counts = np.array(workload.CONFIGS[cfg]["counts"], np.float64)
    L = len(counts)
    ln = frames[0][1].cpu().numpy()
    lv = np.minimum(ln[ln >= 1], L) - 1
    share = np.bincount(lv, minlength=L) / max(len(lv), 1)
    return 0.5 * share + 0.5 * counts / counts.sum()


class Timer:
    """CUDA-event time of `steps` frames on `stream`, barrier + synchronize on both sides, max
    over ranks (the recipe's multi-GPU rule)."""

    def __init__(self, dev, world):
        import torch
        self.torch, self.dev, self.world = torch, dev, world

    def barrier(self):
        import torch.distributed as dist
        if self.world > 1:
            dist.barrier()
        self.torch.cuda.synchronize(self.dev)

    def run(self, fn, steps, stream):
        import torch.distributed as dist
        torch = self.torch
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        self.barrier()
        e0.record(stream)
        with torch.cuda.stream(stream):
            for k in range(steps):
                fn(k)
        e1.record(stream)
        self.barrier()
        ms = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device=self.dev)
        if self.world > 1:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        return float(ms.item())


def build_cache(gsc, cfg, dev, local, args, rank, world, mode, frames, S_local):
    import torch
    c = workload.CONFIGS[cfg]
    pos, alb = workload.init_cloud(cfg)
    cache = gsc.GSCache(c["counts"], torch.from_numpy(pos).to(dev), torch.from_numpy(alb).to(dev),
                        seed=cfg, device=local, hparams=dict(cell_edge_scale=args.cell_scale))
    if world > 1:
        from paper_2507_19718_b200 import dist as gdist
        uid = gdist.exchange_unique_id()
        if mode == 1:
            cache.set_level_weights(level_weights(cfg, frames))
        cache.set_comm(uid, rank, world, mode)
    cache.reserve(S_local, S_local)
    return cache


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
    strong = args.scaling == "strong"
    MODES = {"dp": 0, "level": 1, "oc": 2, "zero": 3}
    NAMES = {v: k for k, v in MODES.items()}
    mode = MODES[args.parallelism]
    R = 4                                   # rotating frames: inputs of step k last used 4 steps ago
    frames, S = make_frames(cfg, rank, world, R, strong, args.morton, dev)
    in_bytes = sum(t.numel() * t.element_size() for t in frames[0])
    outq = torch.empty((S, 3), dtype=torch.float32, device=dev)
    cache = build_cache(gsc, cfg, dev, local, args, rank, world, mode, frames, S)
    stream = torch.cuda.Stream(device=dev)
    if not args.no_defer:       # each frame's optimizer step overlaps the next frame's ingest
        cache.set_deferred_step(True)
    use_graph = not args.no_graph and not (mode in (1, 2) and world > 1)   # modes 1 and 2 are not capturable
    timer = Timer(dev, world)

    def frame_call(cch, x, ln, rgb, xq, lq, out, s_, separate=args.separate):
        if separate:                        # two calls, serialised on one stream
            cch.query(xq, lq, out=out, stream=s_)
            return cch.fit(x, ln, rgb, stream=s_)
        # one call: the lookups overlap the fit samples' ingest and fwd/bwd (internal stream)
        return cch.fit_query(x, ln, rgb, xq, lq, out=out, stream=s_)[1]

    def step(f, s_):
        return frame_call(cache, *frames[f], outq, s_)

    # warm-up (eager), then capture one CUDA graph per rotating frame
    with torch.cuda.stream(stream):
        for w in range(max(args.warmup, 1)):
            step(w % R, stream)
    stream.synchronize()
    graphs = []
    if use_graph:
        for f in range(R):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                step(f, stream)
            graphs.append(g)
        with torch.cuda.stream(stream):
            for w in range(args.warmup):
                graphs[w % R].replay()
    stream.synchronize()

    def timed(k):
        if graphs:
            graphs[k % R].replay()
        else:
            step(k % R, stream)
        if k == args.steps - 1:
            cache.flush(stream)        # the last frame's deferred step is inside the timed region

    # ---- timed region (device time, CUDA events on the launching stream)
    with Clocks(local) as clk:
        ms_step = timer.run(timed, args.steps, stream)
        if args.clock_window > 0:     # keep the GPU busy long enough for nvidia-smi samples;
            # the same number of frames on every rank (each frame holds collectives)
            rounds = max(1, int(args.clock_window * 1e3 / (ms_step * 20)))
            with torch.cuda.stream(stream):
                for _ in range(rounds):
                    for k in range(20):
                        (graphs[k % R].replay() if graphs else step(k % R, stream))
                    stream.synchronize()
    st = cache._stats
    torch.cuda.synchronize(dev)
    n_valid = int(st.n_valid)           # last step's valid samples, global (summed over ranks)
    value = n_valid / (ms_step * 1e-3)
    S_q_total = S * world

    # ---- the other multi-GPU modes, same frames (N > 1 only)
    def time_mode(alt_mode):
        cache_b = build_cache(gsc, cfg, dev, local, args, rank, world, alt_mode, frames, S)
        if not args.no_defer:
            cache_b.set_deferred_step(True)

        def alt_step(k):
            frame_call(cache_b, *frames[k % R], outq, stream)
            if k == args.steps - 1:
                cache_b.flush(stream)
        with torch.cuda.stream(stream):
            for w in range(args.warmup):
                frame_call(cache_b, *frames[w % R], outq, stream)
        ms_alt = timer.run(alt_step, args.steps, stream)
        nv = int(cache_b._stats.n_valid)
        info = cache_b.comm_info()
        a_ = {"parallelism": NAMES[alt_mode] + str(world), "value": nv / (ms_alt * 1e-3), "ms_per_step": ms_alt,
              "cuda_graph": False, "owned_levels_rank0": info["owned_levels"] if rank == 0 else None}
        if alt_mode == 1:
            a_["plan"] = gsc.level_plan(list(level_weights(cfg, frames)), world)
        return a_

    alt = None
    if world > 1 and not args.no_alt:
        alt = []
        for alt_mode in (m for m in (0, 1, 2, 3) if m != mode):
            try:                              # a failing alternative mode is reported, not fatal
                alt.append(time_mode(alt_mode))
            except Exception as e:
                alt.append({"parallelism": NAMES[alt_mode] + str(world), "error": str(e)[:300]})

    # ---- per-kernel device time of the same steps, eager with events per kernel, the two
    # halves serialised (gc_query + gc_fit) so that no kernel's time includes an overlap
    cache.set_deferred_step(False)
    cache.flush(stream)
    cache.profile_enable(True)
    cache.profile_read(reset=True)
    ms_eager = timer.run(lambda k: frame_call(cache, *frames[k % R], outq, stream, separate=True),
                         args.steps, stream)
    prof = cache.profile_read(reset=True)
    cache.profile_enable(False)
    cache.set_deferred_step(not args.no_defer)
    launches_per_step = sum(v[1] for v in prof.values()) / args.steps
    kernel_ms = {k: v[0] / max(v[1], 1) for k, v in prof.items()}
    share = {k: v[0] / args.steps / ms_eager for k, v in prof.items()}
    top = max(prof, key=lambda k: prof[k][0])
    n_pairs, n_cand = int(st.n_pairs), int(st.n_candidates)
    pk, pk_kind = peaks()
    traffic_all, traffic_src = {}, None
    try:   # per-launch DRAM bytes of each kernel from the committed ncu launch list
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        traffic_all = {k.split("::")[-1].split("<")[0]: v for k, v in tj["bytes_per_launch"].items()}
        traffic_src = "profiles/traffic.json: " + tj["source"]
    except Exception:
        pass
    kmap = {"fwdbwd": "k_fwdbwd", "query_fwd": "k_query", "ingest_keys": "k_keys", "query_keys": "k_keys",
            "ingest_scatter": "k_scatter", "query_scatter": "k_scatter", "scan": "k_scan",
            "cull_emit": "k_cull_emit", "record_cull": "k_record_cull", "adamw": "k_adamw", "stats": "k_stats"}
    traffic = traffic_all.get(kmap.get(top, "k_" + top))
    issue_all = {}
    try:   # issue rate / pipe utilisation per kernel from the committed ncu capture
        with open(os.path.join(ROOT, "profiles", "issue.json")) as f:
            ij = json.load(f)
        issue_all, issue_src = ij["kernels"], "profiles/issue.json: " + ij["source"]
    except Exception:
        issue_src = None
    per_kernel = {}
    for k, ms_k in kernel_ms.items():
        kk = kmap.get(k, "k_" + k)
        e = {"ms": ms_k}
        if kk in traffic_all and ms_k > 0:
            gbs = traffic_all[kk] / (ms_k * 1e-3) / 1e9
            e.update(dram_gbs=gbs, dram_frac=gbs / pk["hbm_gbs"])
        if kk in issue_all:
            e.update(ipc=issue_all[kk]["ipc"], issue_frac=issue_all[kk]["ipc"] / 4.0)
        per_kernel[k] = e
    issue = None
    if "k_" + top in issue_all:
        m = issue_all["k_" + top]
        issue = {"ipc": m["ipc"], "peak_ipc": 4.0, "frac": m["ipc"] / 4.0, "fma_pipe_pct": m["fma_pipe_pct"],
                 "xu_pipe_pct": m["xu_pipe_pct"], "source": issue_src}
    n_valid_local = n_valid / world
    pairs_local = n_pairs / world
    if top == "fwdbwd":
        flops = pairs_local * FLOPS_PER_PAIR + n_valid_local * FLOPS_PER_SAMPLE
        achieved = flops / (kernel_ms[top] * 1e-3) / 1e12
        roof = {"bound": "alu", "achieved": achieved, "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP32_PEAK_TFLOPS, "traffic": traffic, "kernel": top,
                "traffic_source": traffic_src,
                "peak_source": "derived: 148 SM x 128 FP32 lanes x 2 x 1.965 GHz (B200_PROFILING.md counts/clock)",
                "algorithmic": f"{FLOPS_PER_PAIR:.0f} flop/contributing pair + {FLOPS_PER_SAMPLE:.0f}/sample",
                "issue_bound": issue}
    else:
        roof = {"bound": "hbm", "achieved": None, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": None, "traffic": traffic, "kernel": top}
    # whole-step roofline: algorithmic bytes 28/fit sample + 336/Gaussian +
    # 28/lookup and flops 67/pair + 20/sample + 30/lookup pair (lookup pairs at the fit's P)
    G = sum(counts)
    pbar = n_pairs / max(n_valid, 1)
    step_bytes = S * 28 + G * 336 + S * 28
    step_flops = pairs_local * FLOPS_PER_PAIR + n_valid_local * FLOPS_PER_SAMPLE + S * pbar * FLOPS_PER_QPAIR
    t_hbm = step_bytes / (pk["hbm_gbs"] * 1e9)
    t_alu = step_flops / (FP32_PEAK_TFLOPS * 1e12)
    roof["step"] = {"bytes": step_bytes, "flops": step_flops, "t_hbm_us": t_hbm * 1e6, "t_alu_us": t_alu * 1e6,
                    "bound": "hbm" if t_hbm >= t_alu else "alu",
                    "frac": max(t_hbm, t_alu) / (ms_step * 1e-3 / (1 if world == 1 else 1)),
                    "per_gpu": True,
                    "note": "max(B/BW, F/peak) / measured ms_per_step, per GPU; lookup pairs at the fit's mean P"}
    roof["per_kernel"] = per_kernel

    # ---- end to end through the public API with pinned HOST buffers
    hx = [tuple(t.cpu().pin_memory() for t in fr) for fr in frames]
    hout = torch.empty((S, 3), dtype=torch.float32).pin_memory()
    with torch.cuda.stream(stream):
        for w in range(2):
            frame_call(cache, *hx[w % R], hout, stream)

    def e2e_step(k):
        frame_call(cache, *hx[k % R], hout, stream)
        if k == args.steps - 1:
            cache.flush(stream)
    ms_e2e = timer.run(e2e_step, args.steps, stream)
    e2e_val = n_valid / (ms_e2e * 1e-3)

    # ---- screen-space path (next row f1): gc_render of all levels and gc_fit_image on one
    # 1920 x 1080 frame of per-level radiance images, rank 0 at N = 1, on a separate cache
    screen = None
    if rank == 0 and world == 1 and not args.no_screen:
        screen = screen_bench(gsc, cfg, dev, local, args)

    # ---- the general path (rotated anisotropic Gaussians, scale LR > 0: the non-lite backward
    # with the Cholesky test and the full dA chain), same frames and frame call, rank 0 at N = 1
    general = None
    if rank == 0 and world == 1 and not args.no_general:
        general = general_bench(gsc, cfg, dev, local, args, frames, S, outq, stream, frame_call)

    # ---- row A8: dense all-pairs lookups, tensor cores vs the CUDA-core evaluator (rank 0, N = 1)
    dense = None
    if rank == 0 and world == 1 and not args.no_dense:
        dense = dense_bench(gsc, dev, local, args)

    # ---- CPU oracle baseline (rank 0, N = 1 only), bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cache, cfg, args.cpu_samples or S)

    if rank == 0:
        line = {
            "metric": metric_name(cfg), "value": value, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": c["name"], "levels": len(counts), "counts": counts,
                       "S_fit_per_gpu": S, "S_query_per_gpu": S,
                       "S_fit_global": S * world,
                       "parallelism": NAMES[mode] + str(world),
                       "l2": f"{R} rotating device-resident frames ({R * in_bytes / 1e6:.0f} MB) > 126 MB L2",
                       "cuda_graph": bool(graphs),
                       "frame_call": "gc_query + gc_fit" if args.separate else "gc_fit_query",
                       "deferred_step": not args.no_defer,
                       "sample_order": "morton" if args.morton else "random"},
            "queries_per_s": S_q_total / (ms_step * 1e-3),
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
        if alt:
            line["alt"] = alt
        if general:
            line["general"] = general
        if screen:
            line["screen"] = screen
        if dense:
            line["dense_a8"] = dense
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def general_bench(gsc, cfg, dev, local, args, frames, S, outq, stream, frame_call):
    """The headline frame on the general path: every level of the config's cache rotated and
    anisotropic (random quaternions, log-scales + U(-0.4, 0.2)), scale LR 0.0125 (the paper's
    -CO variant), so the non-lite kernels run (9-FMA Cholesky test, the 12-term dA
    backward, the scale group in AdamW); same frames, frame call, deferred step and CUDA
    graphs as the headline; device time with CUDA events."""
    import torch
    c = workload.CONFIGS[cfg]
    pos, alb = workload.init_cloud(cfg)
    hp = gsc.default_hparams(lr=[1.16e-3, 1e-3, 1.25e-2, 1.25e-2, 1.5e-1], cell_edge_scale=args.cell_scale)
    cache = gsc.GSCache(c["counts"], torch.from_numpy(pos).to(dev), torch.from_numpy(alb).to(dev),
                        seed=cfg, device=local, hparams=hp)
    r = np.random.default_rng(31)
    for l in range(len(c["counts"])):
        Pl = cache.params_rows(l)
        Pl[:, 3:7] = r.normal(size=(len(Pl), 4)).astype(np.float32)
        Pl[:, 10:13] += r.uniform(-0.4, 0.2, (len(Pl), 3)).astype(np.float32)
        cache.set_params_rows(l, Pl)
    cache.reserve(S, S)
    if not args.no_defer:
        cache.set_deferred_step(True)
    R = len(frames)
    with torch.cuda.stream(stream):
        for w in range(max(args.warmup, 1)):
            frame_call(cache, *frames[w % R], outq, stream)
    stream.synchronize()
    graphs = []
    if not args.no_graph:
        for f in range(R):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                frame_call(cache, *frames[f], outq, stream)
            graphs.append(g)
    n = max(5, args.steps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        for w in range(args.warmup):
            (graphs[w % R].replay() if graphs else frame_call(cache, *frames[w % R], outq, stream))
        e0.record(stream)
        for k in range(n):
            (graphs[k % R].replay() if graphs else frame_call(cache, *frames[k % R], outq, stream))
        cache.flush(stream)
        e1.record(stream)
    stream.synchronize()
    ms = e0.elapsed_time(e1) / n
    st = cache._stats
    nv = int(st.n_valid)
    return {"ms_per_step": ms, "value": nv / (ms * 1e-3), "unit": "samples/s",
            "pairs_per_sample": int(st.n_pairs) / max(nv, 1),
            "candidates_per_sample": int(st.n_candidates) / max(nv, 1),
            "cuda_graph": bool(graphs),
            "workload": c["name"] + ", every level rotated + anisotropic, scale LR 0.0125 (non-lite path)"}


def screen_bench(gsc, cfg, dev, local, args, W=1920, H=1080):
    """gc_render (all levels, one joint raster) and gc_fit_image (render + Eq. 4 + backward +
    AdamW + culling rebuild) on the config's cache at 1920 x 1080; CUDA events on the calling
    stream (each call synchronises the host once to size its sort)."""
    import torch
    c = workload.CONFIGS[cfg]
    pos, alb = workload.init_cloud(cfg)
    cache = gsc.GSCache(c["counts"], torch.from_numpy(pos).to(dev), torch.from_numpy(alb).to(dev),
                        seed=cfg, device=local)
    from scipy.spatial.transform import Rotation
    view = np.hstack([Rotation.from_rotvec([0.15, -0.2, 0.05]).as_matrix(), [[0.02], [-0.03], [3.0]]])
    cam = gsc.make_camera(W, H, 1400.0, 1470.0, W / 2, H / 2, view)
    L = len(c["counts"])
    r = np.random.default_rng(0)
    tgt = torch.from_numpy(r.uniform(0, 1, (L, H, W, 3)).astype(np.float32)).to(dev)
    valid = torch.from_numpy((r.random((L, H, W)) < 0.5).astype(np.uint8)).to(dev)
    s = torch.cuda.current_stream(dev)
    for _ in range(2):
        cache.render(cam)
        cache.fit_image(cam, tgt, valid)
    torch.cuda.synchronize(dev)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    n = max(3, args.steps // 4)
    e[0].record(s)
    for _ in range(n):
        cache.render(cam)
    e[1].record(s)
    e[2].record(s)
    for _ in range(n):
        cache.fit_image(cam, tgt, valid)
    e[3].record(s)
    torch.cuda.synchronize(dev)
    ms_r, ms_f = e[0].elapsed_time(e[1]) / n, e[2].elapsed_time(e[3]) / n
    st = cache._stats
    return {"image": [W, H], "levels": L, "render_ms": ms_r, "fit_image_ms": ms_f,
            "pixel_samples_fitted_per_s": int(st.n_valid) / (ms_f * 1e-3),
            "note": "gc_render of all levels in one joint raster; gc_fit_image = render + Eq. 4 + "
                    "backward + AdamW + culling rebuild; valid pixels 50 % per level"}


def dense_bench(gsc, dev, local, args, S=262_144):
    """Row A8 on the dense case it is meant for: configs[1]'s 3 levels (4096/1024/256) with
    tau = infinity (every Gaussian of a level contributes to every lookup) and a rotated
    anisotropic level 0; 262,144 lookups per call.  gc_query_dense (tcgen05 3xTF32 Q + CUDA-core
    exp/colour epilogue) vs gc_query (the packed fp32x2 CUDA-core evaluator over the one-cell
    culling lists), device time per call with CUDA events; pairs = sum over lookups of the
    level's Gaussian count; MUFU roofline = one ex2 per pair at 148 x 16 / clk (the fit step:
    two, forward and backward).  Also the fit step on the same case: gc_fit_dense (forward +
    Eq. 4 + the two-product tensor-core backward + AdamW + rebuild) vs gc_fit."""
    import torch
    counts = workload.CONFIGS[1]["counts"]
    pos, alb = workload.init_cloud(1)
    c = gsc.GSCache(counts, torch.from_numpy(pos[:counts[0]]).to(dev), torch.from_numpy(alb[:counts[0]]).to(dev),
                    seed=7, device=local, hparams=dict(cutoff_sigma=float("inf")))
    r = np.random.default_rng(11)
    P0 = c.params_rows(0)
    P0[:, 3:7] = r.normal(size=(len(P0), 4)).astype(np.float32)
    P0[:, 10:13] += r.uniform(-0.3, 0.3, (len(P0), 3)).astype(np.float32)
    c.set_params_rows(0, P0)
    xq, lq = workload.query_batch(1, S=S, frame=1)
    xd, ld = torch.from_numpy(xq).to(dev), torch.from_numpy(lq).to(dev)
    out = torch.empty((S, 3), dtype=torch.float32, device=dev)
    c.reserve(0, S)
    lv = np.minimum(lq, len(counts)) - 1
    pairs = float(sum(np.sum(lv == l) * counts[l] for l in range(len(counts))))
    s = torch.cuda.current_stream(dev)
    res = {}
    # the dense fit step on the same case: gc_fit_dense (tensor-core forward + backward) vs gc_fit
    # (CUDA-core evaluators over the one-cell lists), each with AdamW and the list rebuild
    r2 = np.random.default_rng(12)
    rgbd = torch.from_numpy(r2.uniform(0, 2, (S, 3)).astype(np.float32)).to(dev)
    c.reserve(S, S)
    for name, fn in (("fit_tensor_core", lambda: c.fit_dense(xd, ld, rgbd)),
                     ("fit_cuda_core", lambda: c.fit(xd, ld, rgbd))):
        for _ in range(2):
            fn()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = max(3, args.steps // 4)
        e0.record(s)
        for _ in range(n):
            fn()
        e1.record(s)
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1) / n
        res[name] = {"ms": ms, "pairs_per_s": pairs / (ms * 1e-3)}
    for name, fn in (("tensor_core", lambda: c.query_dense(xd, ld, out=out)),
                     ("cuda_core", lambda: c.query(xd, ld, out=out))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = max(5, args.steps // 2)
        e0.record(s)
        for _ in range(n):
            fn()
        e1.record(s)
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1) / n
        res[name] = {"ms": ms, "pairs_per_s": pairs / (ms * 1e-3)}
    mufu = 148 * 16 * 1.965e9
    for k, v in res.items():
        v["mufu_frac"] = v["pairs_per_s"] / mufu * (2 if k.startswith("fit") else 1)   # fit: 2 ex2 per pair
    res.update(workload="cfg1 levels, tau = inf, rotated anisotropic level 0", lookups=S, pairs=pairs,
               speedup=res["cuda_core"]["ms"] / res["tensor_core"]["ms"],
               fit_speedup=res["fit_cuda_core"]["ms"] / res["fit_tensor_core"]["ms"],
               mufu_peak="148 SM x 16 ex2/clk x 1.965 GHz (one ex2 per pair)")
    return res


# CPU oracle baseline, multi-process leg: the oracle as it stands, one process per core over
# contiguous sample shards (C9: per-shard sums add up; the shards' gradient sums are combined
# with the per-level counts, then one AdamW step), set up before the pool forks.
_MP = {}


def _mp_shard(k):
    import oracle
    d = _MP
    lo, hi = d["fit_cuts"][k], d["fit_cuts"][k + 1]
    qlo, qhi = d["q_cuts"][k], d["q_cuts"][k + 1]
    oracle.query(d["goff"], d["P"], d["xq"][qlo:qhi], d["lq"][qlo:qhi], grids=d["grids"])
    r = oracle.loss_grad(d["goff"], d["P"], d["x"][lo:hi], d["ln"][lo:hi], d["rgb"][lo:hi], grids=d["grids"])
    goff = d["goff"]
    g = r["grad"].copy()
    for l in range(len(goff) - 1):   # back to plain sums: the shard normalised by its own 3 k_l
        g[goff[l]:goff[l + 1]] *= 3.0 * r["count"][l]
    return g, r["count"]


def cpu_baseline(cache, cfg, n):
    """The fp64 oracle on this box's host cores: one fit + query step on a bounded sample of the
    same frame, from the same parameters and culling grids -- single thread (the culled oracle
    as it stands), all cores (one oracle process per core over sample shards), plus the
    brute-force oracle (the definition, no culling) on cfg0 and on a cfg1 sample."""
    import multiprocessing as mp

    import oracle
    P = np.concatenate([cache.params_rows(l) for l in range(cache.L)]).astype(np.float64)
    grids = cache.grids()
    oc = oracle.OracleCache(cache.counts, P.copy(), grids=grids)
    x, ln, rgb = workload.fit_batch(cfg, frame=0, S=n)
    xq, lq = workload.query_batch(cfg, frame=0, S=n)
    x, rgb, xq = x.astype(np.float64), rgb.astype(np.float64), xq.astype(np.float64)
    t0 = time.perf_counter()
    oc.query(xq, lq)
    r = oc.fit(x, ln, rgb)
    dt = time.perf_counter() - t0
    nvalid = int(r["count"].sum())
    info = cpu_info()
    out = {"value": nvalid / dt, "unit": "samples/s", "cores": 1, "kind": "oracle",
           "sample": f"{n} fit samples + {n} queries of {workload.CONFIGS[cfg]['name']} frame 0 "
                     f"(culled fp64 oracle, single thread, {dt:.1f} s)",
           "host": info}
    # all cores
    ncores = max(1, int(info["usable_cores"] or 1))
    try:
        goff = np.concatenate([[0], np.cumsum(cache.counts)]).astype(np.int64)
        _MP.update(goff=goff, P=P, grids=grids, x=x, ln=ln, rgb=rgb, xq=xq, lq=lq,
                   fit_cuts=np.linspace(0, n, ncores + 1).astype(np.int64),
                   q_cuts=np.linspace(0, n, ncores + 1).astype(np.int64))
        ctx = mp.get_context("fork")
        with ctx.Pool(ncores) as pool:
            pool.map(_mp_shard, range(ncores))              # warm (fork, library load)
            t0 = time.perf_counter()
            parts = pool.map(_mp_shard, range(ncores))
            gsum = sum(p[0] for p in parts)
            cnt = sum(p[1] for p in parts)
            Pm = P.copy()
            M, V = np.zeros_like(Pm), np.zeros_like(Pm)
            for l in range(len(goff) - 1):
                if cnt[l] > 0:
                    gsum[goff[l]:goff[l + 1]] /= 3.0 * cnt[l]
            oracle.adamw(Pm, M, V, gsum, 1e-3, 1e-2, 0.9, 0.999, 1e-8, 1)   # one step's AdamW work
            dtm = time.perf_counter() - t0
        out["all_cores"] = {"value": nvalid / dtm, "cores": ncores, "seconds": dtm}
    except Exception as e:   # report, do not hide
        out["all_cores"] = {"error": str(e)[:200]}
    # brute force (no culling): cfg0 full step, cfg1 on a bounded sample
    try:
        c0 = workload.CONFIGS[0]
        pos0, rgb0, ls0 = workload.cfg0_lattice()
        P0 = oracle.create(c0["counts"], pos0.astype(np.float64), rgb0.astype(np.float64),
                           ls0.astype(np.float64), seed=0)
        xs, ls = workload.cfg0_samples(c0["S"])
        t0 = time.perf_counter()
        oracle.loss_grad([0, 64], P0, xs.astype(np.float64), ls, np.ones((len(xs), 3)))
        b0 = time.perf_counter() - t0
        c1 = workload.CONFIGS[1]
        pos1, alb1 = workload.init_cloud(1)
        P1 = oracle.create(c1["counts"], pos1.astype(np.float64), alb1.astype(np.float64), seed=1)
        n1 = 8192
        x1, l1, r1 = workload.fit_batch(1, frame=0, S=n1)
        goff1 = np.concatenate([[0], np.cumsum(c1["counts"])])
        t0 = time.perf_counter()
        r1o = oracle.loss_grad(goff1, P1, x1.astype(np.float64), l1, r1.astype(np.float64))
        b1 = time.perf_counter() - t0
        out["brute_force"] = {"cfg0_step_s": b0, "cfg0_samples_per_s": c0["S"] / b0,
                              "cfg1_samples_per_s": int(r1o["count"].sum()) / b1,
                              "cfg1_sample": f"{n1} samples of cfg1 frame 0, every Gaussian of the level",
                              "cores": 1}
    except Exception as e:
        out["brute_force"] = {"error": str(e)[:200]}
    return out


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
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--parallelism", default="dp", choices=["dp", "level", "oc", "zero"],
                    help="dp: data parallel (mode 0); level: level-sharded (mode 1); oc: spatial owner-computes "
                         "(mode 2); zero: data parallel with a reduce-scattered, sharded optimizer (mode 3)")
    ap.add_argument("--no-alt", action="store_true", help="N > 1: do not also time the other mode")
    ap.add_argument("--no-screen", action="store_true", help="skip the screen-space (f1) timing")
    ap.add_argument("--no-dense", action="store_true", help="skip the dense tensor-core (A8) timing")
    ap.add_argument("--no-general", action="store_true",
                    help="skip the general-path (anisotropic, scale LR > 0) timing")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args.gpus)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

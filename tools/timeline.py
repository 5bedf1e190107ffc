"""Kernel timeline of a few bench frames (torch.profiler / CUPTI): start, end, stream per kernel.

  python tools/timeline.py [--config 2] [--frames 3] [--graph] > gpurun_out/timeline.txt
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_19718_b200 as gsc  # noqa: E402
import workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--frames", type=int, default=3)
ap.add_argument("--graph", action="store_true")
ap.add_argument("--no-defer", action="store_true")
args = ap.parse_args()
cfg = workload.CONFIGS[args.config]
pos, alb = workload.init_cloud(args.config)
dev = torch.device("cuda", 0)
cache = gsc.GSCache(cfg["counts"], torch.from_numpy(pos).to(dev), torch.from_numpy(alb).to(dev), seed=args.config)
S = cfg["S"]
frames = []
for f in range(2):
    x, ln, rgb = workload.fit_batch(args.config, frame=f)
    xq, lq = workload.query_batch(args.config, frame=f)
    frames.append(tuple(torch.from_numpy(a).to(dev) for a in (x, ln, rgb, xq, lq)))
out = torch.empty((S, 3), device=dev)
cache.reserve(S, S)
if not args.no_defer:
    cache.set_deferred_step(True)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for w in range(4):
        cache.fit_query(*frames[w % 2], out=out, stream=st)
torch.cuda.synchronize()
graphs = []
if args.graph:
    for f in range(2):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            cache.fit_query(*frames[f], out=out, stream=st)
        graphs.append(g)
    with torch.cuda.stream(st):
        for w in range(2):
            graphs[w % 2].replay()
    torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    with torch.cuda.stream(st):
        for k in range(args.frames):
            if graphs:
                graphs[k % 2].replay()
            else:
                cache.fit_query(*frames[k % 2], out=out, stream=st)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
rows = []
for e in ev:
    t0 = e.time_range.start
    rows.append((t0, e.time_range.end, getattr(e, "stream", -1) if hasattr(e, "stream") else -1, e.name))
rows.sort()
base = rows[0][0] if rows else 0
for t0, t1, s, n in rows:
    print(f"{(t0 - base):9.1f} {(t1 - base):9.1f} {t1 - t0:7.1f}  {str(s):>4}  {n[:60]}")

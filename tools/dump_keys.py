"""Dump cfg2 fit-sample cell keys (computed with numpy from gc_grid) for tools/microbench_atomics."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2507_19718_b200 as gsc, workload
pos, alb = workload.init_cloud(2)
c = gsc.GSCache(workload.CONFIGS[2]["counts"], torch.from_numpy(pos).cuda(), torch.from_numpy(alb).cuda(), seed=2)
x, ln, rgb = workload.fit_batch(2)
L = c.L
coff = [0]
keys = np.full(len(x), 0xFFFFFFFF, np.uint64)
for l in range(L):
    o, ic, d = c.grid(l)
    coff.append(coff[-1] + int(np.prod(d)))
lvl = np.minimum(ln, L) - 1
for l in range(L):
    o, ic, d = c.grid(l)
    m = lvl == l
    cc = np.clip(np.floor((x[m].astype(np.float64) - o) * ic), 0, d - 1).astype(np.int64)
    keys[m] = coff[l] + (cc[:, 2] * d[1] + cc[:, 1]) * d[0] + cc[:, 0]
keys = keys[lvl >= 0].astype(np.uint32)
print("n", len(keys), "cells", coff[-1], "max per cell", np.bincount(keys).max())
keys.tofile("gpurun_out/keys_cfg2.bin")
open("gpurun_out/keys_cfg2.txt", "w").write(f"{len(keys)} {coff[-1]}\n")

"""Work-item statistics of a cfg frame (lane utilisation of the evaluators): per level, cells,
items, useful tests (sum count*C) vs lane-slot tests (sum slots*C, slots 32 or 64).

  python tools/item_stats.py [--config 2] [--cell-scale 1.0]
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2507_19718_b200 as gsc, workload

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--ch", type=int, default=64)
args = ap.parse_args()
pos, alb = workload.init_cloud(args.config)
c = gsc.GSCache(workload.CONFIGS[args.config]["counts"], torch.from_numpy(pos).cuda(),
                torch.from_numpy(alb).cuda(), seed=args.config)
L = c.L
for name, (x, ln) in (("fit", workload.fit_batch(args.config)[:2]), ("query", workload.query_batch(args.config))):
    lvl = np.minimum(ln, L) - 1
    tot_u = tot_s = tot_items = 0
    hist = np.zeros(65, np.int64)
    for l in range(L):
        o, ic, d = c.grid(l)
        off, _ = c.debug_cull(l)
        Cc = np.diff(off.astype(np.int64))
        m = lvl == l
        cc = np.clip(np.floor((x[m].astype(np.float64) - o) * ic), 0, d - 1).astype(np.int64)
        key = (cc[:, 2] * d[1] + cc[:, 1]) * d[0] + cc[:, 0]
        n = np.bincount(key, minlength=len(Cc))
        nz = n > 0
        n, Cn = n[nz], Cc[nz]
        full, rem = n // args.ch, n % args.ch
        items = full + (rem > 0)
        slots = full * 64 + np.where(rem > 32, 64, np.where(rem > 0, 32, 0))
        u, s = int((n * Cn).sum()), int((slots * Cn).sum())
        hist += np.bincount(np.minimum(rem[rem > 0], 64), minlength=65)[:65]
        hist[args.ch] += int(full.sum())
        print(f"{name} L{l}: samples {int(n.sum())} cells {int(nz.sum())} items {int(items.sum())} "
              f"mean n/cell {n.mean():.1f} C(w) {u / max(1, n.sum()):.1f} util {u / max(1, s):.3f}")
        tot_u += u; tot_s += s; tot_items += int(items.sum())
    print(f"{name}: items {tot_items} useful tests {tot_u/1e6:.1f} M slot tests {tot_s/1e6:.1f} M util {tot_u/tot_s:.3f}")
    q = np.cumsum(hist) / hist.sum()
    print(f"{name}: item count quantiles  <=8 {q[8]:.2f} <=16 {q[16]:.2f} <=32 {q[32]:.2f} <=48 {q[48]:.2f}")

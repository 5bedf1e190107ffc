"""Minimal eager cfg2 fit+query step driver for ncu captures (no timing is reported)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_19718_b200 as gsc  # noqa: E402
import workload  # noqa: E402

cfg = int(os.environ.get("CFG", "2"))
steps = int(os.environ.get("STEPS", "3"))
c = workload.CONFIGS[cfg]
pos, alb = workload.init_cloud(cfg)
cache = gsc.GSCache(c["counts"], torch.from_numpy(pos).cuda(), torch.from_numpy(alb).cuda(), seed=cfg)
x, ln, rgb = (torch.from_numpy(a).cuda() for a in workload.fit_batch(cfg))
xq, lq = (torch.from_numpy(a).cuda() for a in workload.query_batch(cfg))
out = torch.empty((len(xq), 3), device="cuda")
for _ in range(steps):
    cache.query(xq, lq, out=out)
    st = cache.fit(x, ln, rgb)
torch.cuda.synchronize()
print("ok", st.n_valid, st.n_pairs, st.n_candidates)

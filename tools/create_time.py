"""gc_create wall time at cfg2 / cfg4 (Eq. 2 3-NN, records, culling lists): python tools/create_time.py
Each config is created three times; the first includes lazy module loading, the best is reported."""
import time, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2507_19718_b200 as gsc, workload
for cfg in (2, 4):
    pos, alb = workload.init_cloud(cfg)
    P, A = torch.from_numpy(pos).cuda(), torch.from_numpy(alb).cuda()
    ts = []
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        c = gsc.GSCache(workload.CONFIGS[cfg]["counts"], P, A, seed=cfg)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
        del c
    print(f"cfg{cfg} create {min(ts):.3f} s (runs {', '.join(f'{x:.3f}' for x in ts)}; G = "
          f"{sum(workload.CONFIGS[cfg]['counts'])})", flush=True)

"""Small end-to-end case for compute-sanitizer (memcheck / racecheck / synccheck): cfg0 and a
reduced cfg1 through every hot-path call (create, fit, query, fit_query with the Eq. 3
epilogue, deferred step + flush, gc_params, Alg. 1 batch).  Exits 0 when the calls succeed."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2507_19718_b200 as gsc  # noqa: E402
import workload  # noqa: E402


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def main():
    pos, rgb, ls = workload.cfg0_lattice()
    c0 = gsc.GSCache([64], cu(pos), cu(rgb), init_log_scale=cu(ls))
    x, ln = workload.cfg0_samples(4096)
    y = np.ones((4096, 3), np.float32)
    for _ in range(3):
        c0.fit(cu(x), cu(ln), cu(y))
    c0.query(cu(x), cu(ln))
    pos1, alb1 = workload.init_cloud(1)
    c1 = gsc.GSCache([4096, 1024, 256], cu(pos1[:4096]), cu(alb1[:4096]), seed=7)
    xf, lf, rf = workload.fit_batch(1, S=20_000, frame=1)
    xq, lq = workload.query_batch(1, S=20_000, frame=1)
    c1.fit(cu(xf), cu(lf), cu(rf))
    c1.set_deferred_step(True)
    for f in range(2):
        c1.fit_query(cu(xf), cu(lf), cu(rf), cu(xq), cu(lq), attenuation=cu(np.full((20_000, 3), 0.5, np.float32)))
    c1.flush()
    c1.params_rows(0)
    sig = cu(np.random.default_rng(0).uniform(0, 1, (1000, 4, 3)).astype(np.float32))
    gsc.alg1_terminate(sig, cu(np.full(1000, 3, np.int32)), 1.0, cu(np.random.default_rng(1).random(1000).astype(np.float32)))
    torch.cuda.synchronize()
    print("sanitize case ok")


if __name__ == "__main__":
    main()

"""Multi-rank worker of tests/test_multi_gpu.py (launched by torchrun, one rank per GPU).

Every rank holds the same cfg1 cache and passes its own contiguous shard of one global batch;
after one gc_fit_query + one gc_fit the N-rank result must equal the one-rank oracle on the
concatenated batch (C9): per-level k_l and losses, the first AdamW step (the criterion of
test_first_step_matches_oracle_update), and every lookup in caller order (gathered to rank 0).
Exit status 0 = parity held on every rank.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
import paper_2507_19718_b200 as gsc  # noqa: E402
import workload  # noqa: E402
from paper_2507_19718_b200 import dist as gdist  # noqa: E402


def main():
    mode = int(sys.argv[1])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("gloo")
    counts = [4096, 1024, 256]
    pos, alb = workload.init_cloud(1)
    c = gsc.GSCache(counts, torch.from_numpy(pos).to(dev), torch.from_numpy(alb).to(dev), seed=7, device=local)
    P0 = np.concatenate([c.params_rows(l) for l in range(3)]).astype(np.float64)
    uid = gdist.exchange_unique_id()
    c.set_comm(uid, rank, world, mode)
    x, ln, rgb = workload.fit_batch(1, S=120_000, frame=11)
    xq, lq = workload.query_batch(1, S=40_000, frame=12)
    lo, hi = gdist.shard_range(len(x), rank, world)
    qlo, qhi = gdist.shard_range(len(xq), rank, world)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    y, st = c.fit_query(cu(x[lo:hi]), cu(ln[lo:hi]), cu(rgb[lo:hi]), cu(xq[qlo:qhi]), cu(lq[qlo:qhi]))
    torch.cuda.synchronize()
    ys = [None] * world
    dist.all_gather_object(ys, y.cpu().numpy())
    P1 = np.concatenate([c.params_rows(l) for l in range(3)]).astype(np.float64)   # collective in mode 1
    ok = True
    if rank == 0:
        grids = c.grids()
        oc = oracle.OracleCache(counts, P0, grids=grids)
        yo = oc.query(xq.astype(np.float64), lq)
        yg = np.concatenate(ys)
        err = np.abs(yg - yo) - (1e-5 * np.abs(yo) + 1e-7 * np.abs(yo).max())
        n_bad = int((err > 0).any(axis=1).sum())
        ok &= n_bad <= max(3, int(1e-4 * len(yo)))
        r = oc.fit(x.astype(np.float64), ln, rgb.astype(np.float64))
        for l in range(3):
            ok &= st.count[l] == r["count"][l]
            ok &= abs(st.loss[l] - r["loss"][l]) <= 1e-4 * r["loss"][l]
        go = r["grad"]
        eta = np.array([1.16e-3] * 3 + [1e-3] * 4 + [1.25e-2] * 3 + [0.0] * 3 + [1.5e-1])
        strong = np.abs(go) > 1e-3 * np.abs(go).max(axis=0, keepdims=True)
        e2 = np.abs((P1 - P0) - (oc.P - P0))
        ok &= bool(np.all(e2[strong] <= 1e-3 * eta[np.nonzero(strong)[1]] + 4e-7 * (1 + np.abs(P0[strong]))))
        ok &= bool(np.all(e2 <= 2.0 * eta[None, :] + 4e-7 * (1 + np.abs(P0))))
        print(f"mode {mode} world {world}: lookups off-bar {n_bad}, counts {list(st.count[:3])} "
              f"vs {list(r['count'])}, ok={ok}", flush=True)
    st2 = c.fit(cu(x[lo:hi]), cu(ln[lo:hi]), cu(rgb[lo:hi]))
    torch.cuda.synchronize()
    ok &= st2.step == 2
    flag = torch.tensor([1 if ok else 0])
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 1 else 1)


if __name__ == "__main__":
    main()

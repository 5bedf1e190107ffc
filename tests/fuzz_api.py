"""Randomised API soak on one GPU: random sequences of the public calls (fit, query, fit_query
with and without the deferred step, dense lookups and fits, screen render / fit, parameter and
Adam-state round trips, reinit) on caches of random sizes, inputs of random sizes (including 0)
with dropped samples mixed in; after every call the sticky error state is checked, and every
few calls a query is compared against the fp64 oracle on the library's current parameters.
  python tests/fuzz_api.py [--calls 300] [--seed 0]   (test infrastructure: it calls the oracle;
  tests/test_gpu_fuzz.py runs a short sequence under pytest -m gpu)"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure: checking, not the product path)
import paper_2507_19718_b200 as gsc  # noqa: E402

dev = torch.device("cuda", 0)


r = np.random.default_rng(0)


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def new_cache():
    L = int(r.integers(1, 4))
    n0 = int(r.integers(8, 3000))
    counts = [max(1, n0 >> (2 * l)) for l in range(L)]
    counts = sorted(counts, reverse=True)
    pos = r.uniform(-1, 1, (n0, 3)).astype(np.float32)
    alb = r.uniform(0, 1, (n0, 3)).astype(np.float32)
    tau = float(r.choice([3.0, 3.0, np.inf]))
    c = gsc.GSCache(counts, cu(pos), cu(alb), seed=int(r.integers(0, 100)), hparams=dict(cutoff_sigma=tau))
    return c, counts, tau


def samples(S, L):
    x = r.uniform(-1.2, 1.2, (S, 3)).astype(np.float32)
    ln = r.integers(-1, L + 2, S).astype(np.int32)
    rgb = r.uniform(0, 3, (S, 3)).astype(np.float32)
    if S:
        x[r.random(S) < 0.02] = np.nan
        rgb[r.random(S) < 0.02] = np.inf
    return x, ln, rgb


def check_query(c, counts, tau):
    S = int(r.integers(1, 500))
    x, ln, _ = samples(S, len(counts))
    y = c.query(cu(x), cu(ln)).cpu().numpy()
    P = np.concatenate([c.params_rows(l) for l in range(c.L)]).astype(np.float64)
    yo, lv, _ = oracle.query(c.goff, P, x.astype(np.float64), ln, tau=tau,
                             grids=None if not np.isfinite(tau) else c.grids())
    ok = lv >= 0
    err = np.abs(y[ok] - yo[ok]) / (np.abs(yo[ok]) + 1e-6 * max(np.abs(yo).max(), 1e-30))
    return float(err.max()) if err.size else 0.0


def run(calls=300, seed=0):
    """The soak itself: returns the per-op call counts and the worst relative query error."""
    global r
    from scipy.spatial.transform import Rotation
    r = np.random.default_rng(seed)
    c, counts, tau = new_cache()
    worst, n_calls = 0.0, {}
    for i in range(calls):
        op = r.choice(["fit", "query", "fit_query", "defer", "dense_q", "dense_fit", "render", "fit_image",
                       "params", "adam", "reinit", "new"])
        n_calls[op] = n_calls.get(op, 0) + 1
        L = len(counts)
        S = int(r.choice([0, 1, 7, 129, 1000, 5000]))
        x, ln, rgb = samples(S, L)
        if op == "fit":
            c.fit(cu(x), cu(ln), cu(rgb))
        elif op == "query":
            c.query(cu(x), cu(ln))
        elif op == "fit_query":
            xq, lq, _ = samples(int(r.integers(1, 2000)), L)
            c.fit_query(cu(x), cu(ln), cu(rgb), cu(xq), cu(lq))
        elif op == "defer":
            c.set_deferred_step(bool(r.integers(0, 2)))
        elif op == "dense_q":
            c.query_dense(cu(x), cu(ln))
        elif op == "dense_fit":
            c.fit_dense(cu(x), cu(ln), cu(rgb))
        elif op in ("render", "fit_image"):
            W, H = int(r.integers(1, 120)), int(r.integers(1, 90))
            view = np.hstack([Rotation.from_rotvec(r.normal(0, 0.3, 3)).as_matrix(), [[0.0], [0.0], [float(r.uniform(1.5, 4))]]])
            cam = gsc.make_camera(W, H, float(r.uniform(20, 200)), float(r.uniform(20, 200)), W / 2, H / 2, view)
            if op == "render":
                c.render(cam)
            else:
                tgt = cu(r.uniform(0, 1, (L, H, W, 3)).astype(np.float32))
                va = cu((r.random((L, H, W)) < 0.7).astype(np.uint8))
                c.fit_image(cam, tgt, va)
        elif op == "params":
            l = int(r.integers(0, L))
            P = c.params_rows(l)
            c.set_params_rows(l, P, reset_adam=bool(r.integers(0, 2)))
            assert np.array_equal(c.params_rows(l), P)
        elif op == "adam":
            l = int(r.integers(0, L))
            m, v, ctr = c.adam_state(l)
            c.set_adam_state(l, m, v, ctr)
        elif op == "reinit":
            n0 = counts[0]
            c.reinit(cu(r.uniform(-1, 1, (n0, 3)).astype(np.float32)), cu(r.uniform(0, 1, (n0, 3)).astype(np.float32)))
        elif op == "new":
            c.destroy()
            c, counts, tau = new_cache()
        torch.cuda.synchronize()
        if i % 10 == 9:
            c.flush()
            torch.cuda.synchronize()
            e = check_query(c, counts, tau)
            worst = max(worst, e)
            assert e < 1e-3, (i, op, e)
    return {"calls": calls, "per_op": {str(k): v for k, v in n_calls.items()}, "worst_query_rel_err": worst}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--calls", type=int, default=300)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    print(run(args.calls, args.seed))

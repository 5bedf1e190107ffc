"""Measured parity of the CUDA path against the fp64 oracle (what the -m gpu tests assert,
with the numbers written down; test infrastructure, it calls the oracle):
  python tests/parity_report.py > profiles/r02_parity.json

* forward: cfg1 full frame of lookups -- max relative error per element, samples with an A3
  boundary-ambiguous pair;
* gradients: cfg1, rotated anisotropic level 0, both loss modes -- relative L2 error per
  (level, group);
* culling lists and level assignment: mismatching entries (must be 0);
* 100 fit steps: cfg1 noisy and cfg0 clean -- largest relative loss difference over the curve;
* cfg2 full frame through the bench's frame call: sampled lookups;
* (round 2) screen-space render (all levels, 200 x 150) and fit_image gradients (fp64 central
  differences of the oracle's Eq. 4 image loss); dense tensor-core lookups (gc_query_dense) and
  the dense fit step's gradients (gc_fit_dense) at tau = infinity.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2507_19718_b200 as gsc  # noqa: E402
import workload  # noqa: E402


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def rows(c):
    return np.concatenate([c.params_rows(l) for l in range(c.L)]).astype(np.float64)


def make_cfg1(hp=None):
    pos, alb = workload.init_cloud(1)
    return gsc.GSCache([4096, 1024, 256], cuda(pos), cuda(alb), seed=7, hparams=hp)


def fwd_err(y, yo):
    y, yo = np.asarray(y, np.float64), np.asarray(yo, np.float64)
    rel = np.abs(y - yo) / np.maximum(np.abs(yo), 1e-7 * np.abs(yo).max())
    return float(rel.max()), float(np.median(rel)), int((rel > 1e-5).any(axis=1).sum())


def main():
    out = {}
    # forward
    c = make_cfg1()
    P = rows(c)
    x, ln = workload.query_batch(1)
    y = c.query(cuda(x), cuda(ln)).cpu().numpy()
    yo, lv, _ = oracle.query(c.goff, P, x.astype(np.float64), ln, grids=c.grids())
    mx, med, nbad = fwd_err(y, yo)
    out["forward_cfg1"] = {"points": len(x), "max_rel_err": mx, "median_rel_err": med,
                           "points_over_1e-5": nbad, "tolerance": "1e-5 |y| + 1e-7 max|y| (A3 boundary pairs allowed)"}
    # gradients
    for mode in (0, 1):
        c = make_cfg1(gsc.default_hparams(loss_grad_mode=mode))
        r = np.random.default_rng(6)
        P0 = c.params_rows(0)
        P0[:, 3:7] = r.normal(size=(4096, 4)).astype(np.float32)
        P0[:, 10:13] += r.uniform(-0.3, 0.3, (4096, 3)).astype(np.float32)
        c.set_params_rows(0, P0)
        P = rows(c)
        c.debug_enable_grads(True)
        x, ln, rgb = workload.fit_batch(1)
        st = c.fit(cuda(x), cuda(ln), cuda(rgb))
        torch.cuda.synchronize()
        g = np.concatenate([c.debug_grads_rows(l) for l in range(3)]).astype(np.float64)
        ro = oracle.loss_grad(c.goff, P, x.astype(np.float64), ln, rgb.astype(np.float64), mode=mode, grids=c.grids())
        res = {}
        for l in range(3):
            sl = slice(c.goff[l], c.goff[l + 1])
            for name, cs in oracle.GROUP_SLICES.items():
                a, b = g[sl, cs], ro["grad"][sl, cs]
                if name == "rotation" and l > 0:      # isotropic levels: dq = 0 exactly (the
                    # oracle's fp64 is ~1e-13): report |a| relative to the level's gradient
                    res[f"L{l}/{name} (isotropic, |g|/|g_level|)"] = float(
                        np.linalg.norm(a) / np.linalg.norm(ro["grad"][sl]))
                    continue
                res[f"L{l}/{name}"] = float(np.linalg.norm(a - b) / np.linalg.norm(b))
        out[f"gradients_cfg1_mode{mode}"] = {"rel_l2_err": res, "loss_rel_err": [
            float(abs(st.loss[l] - ro["loss"][l]) / ro["loss"][l]) for l in range(3)], "tolerance": "1e-4"}
    # culling lists, level assignment
    c = make_cfg1()
    P = rows(c)
    bad = 0
    for l in range(3):
        o, ic, d = c.grid(l)
        off_o, idx_o = oracle.csr_for(P[c.goff[l]:c.goff[l + 1]], 3.0, (o, ic, d))
        off_g, idx_g = c.debug_cull(l)
        bad += int((off_g.astype(np.int64) != off_o).sum()) + int((idx_g != idx_o).sum())
    x, ln, rgb = workload.fit_batch(1, S=100_000)
    ln[::17] = 0
    x[::23, 1] = np.nan
    c.fit(cuda(x), cuda(ln), cuda(rgb))
    lg = c.debug_levels(len(x))
    lo = oracle.level_of(ln, 3, x.astype(np.float64), rgb.astype(np.float64))
    out["bit_exact"] = {"culling_list_mismatches": bad, "level_assignment_mismatches": int((lg != lo).sum())}
    # 100-step curves
    c = make_cfg1()
    oc = oracle.OracleCache([4096, 1024, 256], rows(c), grids=c.grids())
    lgc, loc = [], []
    for s in range(100):
        x, ln, rgb = workload.fit_batch(1, frame=s, S=65536)
        st = c.fit(cuda(x), cuda(ln), cuda(rgb))
        torch.cuda.synchronize()
        lgc.append(sum(st.loss[:3]))
        loc.append(oc.fit(x.astype(np.float64), ln, rgb.astype(np.float64))["loss"].sum())
    lgc, loc = np.array(lgc), np.array(loc)
    out["loss_curve_cfg1_100_steps"] = {"max_rel_diff": float((np.abs(lgc - loc) / loc).max()),
                                        "step100_rel_diff": float(abs(lgc[-1] - loc[-1]) / loc[-1]),
                                        "loss_step1": float(loc[0]), "loss_step100": float(loc[-1]), "tolerance": "1 %"}
    # cfg2 frame call (sampled)
    pos, alb = workload.init_cloud(2)
    c = gsc.GSCache(workload.CONFIGS[2]["counts"], cuda(pos), cuda(alb), seed=2)
    c.set_deferred_step(True)
    P = rows(c)
    x, ln, rgb = workload.fit_batch(2)
    xq, lq = workload.query_batch(2)
    y, _ = c.fit_query(cuda(x), cuda(ln), cuda(rgb), cuda(xq), cuda(lq))
    c.flush()
    torch.cuda.synchronize()
    idx = np.random.default_rng(7).choice(len(xq), 3000, replace=False)
    yo, _, _ = oracle.query(c.goff, P, xq[idx].astype(np.float64), lq[idx])
    mx, med, nbad = fwd_err(y.cpu().numpy()[idx], yo)
    out["forward_cfg2_frame_call_sampled"] = {"points": 3000, "max_rel_err": mx, "median_rel_err": med,
                                              "points_over_1e-5": nbad}
    # ---- round 2: screen space (f1)
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import test_gpu_screen as ts
    c = ts.scene(gsc, [1500, 400, 100])
    cam, ocam = ts.camera(gsc, 200, 150, 180.0)
    img = c.render(cam).cpu().numpy()
    P = rows(c)
    errs, namb = [], 0
    for l in range(3):
        yo, _, amb = oracle.render(P[c.goff[l]:c.goff[l + 1]], ocam)
        okp = (amb == 0)
        d = np.abs(img[l] - yo)[okp] / (np.abs(yo)[okp] + 1e-6 * np.abs(yo).max())
        errs.append(float(d.max()))
        namb += int((amb != 0).sum())
    out["screen_render_200x150"] = {"max_rel_err_per_level": errs, "ambiguous_pixels": namb,
                                    "pixels": 3 * 200 * 150, "tolerance": "1e-5 |y| + 1e-6 max|y|"}
    c, cam, ocam, P, target, valid = ts._tiny(gsc)
    c.debug_enable_grads(True)
    c.fit_image(cam, cuda(target.astype(np.float32)), cuda(valid))
    torch.cuda.synchronize()
    g = np.concatenate([c.debug_grads_rows(l) for l in range(2)]).astype(np.float64)
    go = oracle.image_grad_fd(c.goff, P, ocam, target, valid)
    res = {}
    for l in range(2):
        sl = slice(c.goff[l], c.goff[l + 1])
        for name, cs in oracle.GROUP_SLICES.items():
            a, b = g[sl, cs], go[sl, cs]
            res[f"L{l}/{name}"] = float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
    out["screen_fit_image_gradients"] = {"rel_l2_err": res, "reference": "fp64 central differences of the oracle's Eq. 4 image loss"}
    # ---- round 2: dense tensor cores (A8)
    import test_gpu_dense_tc as td
    c = td.dense_cache(gsc, float("inf"), True)
    P = rows(c)
    xq, lq = workload.query_batch(1, S=12_001, frame=6)
    y = c.query_dense(cuda(xq), cuda(lq)).cpu().numpy()
    yo, lv, _ = oracle.query(c.goff, P, xq.astype(np.float64), lq, tau=float("inf"))
    mx, med, nbad = fwd_err(y[lv >= 0], yo[lv >= 0])
    out["dense_tc_lookups_tau_inf"] = {"points": int((lv >= 0).sum()), "max_rel_err": mx, "median_rel_err": med,
                                       "points_over_1e-5": nbad}
    c, x, ln, rgb = td._dense_fit_case(gsc, 1000, 9000, seed=1000)
    P = rows(c)
    c.debug_enable_grads(True)
    st = c.fit_dense(cuda(x), cuda(ln), cuda(rgb))
    torch.cuda.synchronize()
    g = np.concatenate([c.debug_grads_rows(l) for l in range(2)]).astype(np.float64)
    ro = oracle.loss_grad(c.goff, P, x.astype(np.float64), ln, rgb.astype(np.float64), tau=np.inf)
    res = {}
    for l in range(2):
        sl = slice(c.goff[l], c.goff[l + 1])
        for name, cs in oracle.GROUP_SLICES.items():
            a, b = g[sl, cs], ro["grad"][sl, cs]
            if name == "rotation" and l > 0:
                continue
            res[f"L{l}/{name}"] = float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
    out["dense_fit_gradients_tau_inf"] = {"rel_l2_err": res, "loss_rel_err": [
        float(abs(st.loss[l] - ro["loss"][l]) / ro["loss"][l]) for l in range(2)], "tolerance": "1e-4"}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

"""Synthetic analogue of the paper's hyper-parameter ablation (App. A.2, Fig.
'hyperparams'): Ours vs -REG (Adam instead of AdamW: weight decay 0), -CO
(scale LR 0.0125), -CO -REG, and -SC (no Eq. 2 size cap / down-scaling), run through the
library on the GPU.

"Camera" = the half-space of the scene the frame's samples come from: its normal turns a
full circle about z over the first 256 frames (moving viewport), then stays put for 256
(recuperation), as in the paper's protocol.  Reported per variant: held-out relative error
of the lookups against the synthetic truth over all visible structure, averaged over the last
64 frames of each phase, the largest Gaussian extent e^s and the largest |colour|, and
whether anything became non-finite.

  python tools/ablation.py [--config 1] [--frames 256] [--firefly Q] [--screen] > profiles/r01_ablation.json

--screen: the paper's own setting -- the cache is fitted in SCREEN space (gc_fit_image, next
row f1) to noisy per-level radiance images of a camera orbiting the scene once over `frames`
frames, then still for `frames`; error = rendered cache images vs the noise-free images over
the pixels whose primary ray hits the scene.

--firefly Q: the paper's "unpredictably high variance ... gradients [that] can take on large
values, which can occur very sparsely": each sample is additionally multiplied by
F = 300 with probability Q, else by (1 - 300 Q)/(1 - Q) -- still unbiased (E[F] = 1).
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_19718_b200 as gsc  # noqa: E402
import workload  # noqa: E402

VARIANTS = {
    "ours": {},
    "-REG": {"weight_decay": [0.0] * 5},
    "-CO": {"lr_scale": 0.0125},
    "-CO,-REG": {"lr_scale": 0.0125, "weight_decay": [0.0] * 5},
    "-SC": {"init_zcap": 1e30, "init_scale_factor": 1.0},
}


def view_mask(x, theta):
    n = np.array([np.cos(theta), np.sin(theta), 0.0])
    return x @ n > -0.1


def run(cfg, frames, name, over, dev, firefly):
    c = workload.CONFIGS[cfg]
    hp = {}
    if "weight_decay" in over:
        hp["weight_decay"] = over["weight_decay"]
    if "lr_scale" in over:
        lr = [1.16e-3, 1e-3, 1.25e-2, over["lr_scale"], 1.5e-1]
        hp["lr"] = lr
    for k in ("init_zcap", "init_scale_factor"):
        if k in over:
            hp[k] = over[k]
    pos, alb = workload.init_cloud(cfg)
    cache = gsc.GSCache(c["counts"], torch.from_numpy(pos).to(dev), torch.from_numpy(alb).to(dev),
                        seed=cfg, hparams=gsc.default_hparams(**hp))
    L = len(c["counts"])
    S = c["S"] // 2
    xq, lq = workload.query_batch(cfg, frame=99_999, S=100_000)
    lvl_q = np.minimum(lq, L) - 1
    truth = workload.radiance(xq.astype(np.float64), lvl_q)
    xq_d, lq_d = torch.from_numpy(xq).to(dev), torch.from_numpy(lq).to(dev)
    errs, bad = [], False
    for f in range(2 * frames):
        theta = 2 * np.pi * min(f, frames) / frames
        x, ln, rgb = workload.fit_batch(cfg, frame=f, S=2 * S)
        if firefly > 0:
            r = np.random.Generator(np.random.Philox(key=7_000_000 + f))
            hi = r.random(len(rgb)) < firefly
            rgb = (rgb * np.where(hi, 300.0, (1 - 300 * firefly) / (1 - firefly))[:, None]).astype(np.float32)
        m = view_mask(x.astype(np.float64), theta)
        x, ln, rgb = x[m][:S], ln[m][:S], rgb[m][:S]
        st = cache.fit(torch.from_numpy(np.ascontiguousarray(x)).to(dev),
                       torch.from_numpy(np.ascontiguousarray(ln)).to(dev),
                       torch.from_numpy(np.ascontiguousarray(rgb)).to(dev))
        if f % 8 == 7:
            y = cache.query(xq_d, lq_d).cpu().numpy().astype(np.float64)
            vis = view_mask(xq.astype(np.float64), theta)
            e = np.abs(y[vis] - truth[vis]).sum() / max(np.abs(truth[vis]).sum(), 1e-30)
            errs.append((f, float(e)))
            bad = bad or not np.isfinite(y).all() or st.nonfinite_grads > 0
    torch.cuda.synchronize()
    P = np.concatenate([cache.params_rows(l) for l in range(L)])
    e1 = [e for f, e in errs if frames - 64 <= f < frames]
    e2 = [e for f, e in errs if f >= 2 * frames - 64]
    return {"variant": name, "hparams": over,
            "rel_error_moving_last64": float(np.mean(e1)), "rel_error_still_last64": float(np.mean(e2)),
            "max_extent_es": float(np.exp(P[:, 10:13]).max()), "max_abs_colour": float(np.abs(P[:, 7:10]).max()),
            "nonfinite": bool(bad or not np.isfinite(P).all()),
            "curve": errs}


def look_at(theta, dist=3.0, elev=0.35):
    C = dist * np.array([np.cos(theta), np.sin(theta), elev])
    z = -C / np.linalg.norm(C)
    x = np.cross(z, [0.0, 0.0, 1.0])
    x /= np.linalg.norm(x)
    y = np.cross(z, x)
    R = np.stack([x, y, z])
    return np.hstack([R, (-R @ C)[:, None]])


def run_screen(cfg, frames, name, over, dev, W=128, H=96, f=110.0):
    c = workload.CONFIGS[cfg]
    hp = {}
    if "weight_decay" in over:
        hp["weight_decay"] = over["weight_decay"]
    if "lr_scale" in over:
        hp["lr"] = [1.16e-3, 1e-3, 1.25e-2, over["lr_scale"], 1.5e-1]
    for k in ("init_zcap", "init_scale_factor"):
        if k in over:
            hp[k] = over[k]
    pos, alb = workload.init_cloud(cfg)
    cache = gsc.GSCache(c["counts"], torch.from_numpy(pos).to(dev), torch.from_numpy(alb).to(dev),
                        seed=cfg, hparams=gsc.default_hparams(**hp))
    L = len(c["counts"])
    r = np.random.Generator(np.random.Philox(key=4242))
    errs, bad = [], False
    for fr in range(2 * frames):
        theta = 2 * np.pi * min(fr, frames) / frames
        view = look_at(theta)
        cam = gsc.make_camera(W, H, f, f, W / 2, H / 2, view)
        x, hit = workload.primary_hits(view, W, H, f, f, W / 2, H / 2)
        tgt, valid = workload.screen_targets(x, hit, L, r)
        st = cache.fit_image(cam, torch.from_numpy(tgt.astype(np.float32)).to(dev),
                             torch.from_numpy(valid.astype(np.uint8)).to(dev))
        if fr % 8 == 7:
            img = cache.render(cam).cpu().numpy().astype(np.float64)
            xs = np.where(hit[..., None], x, 0.0).reshape(-1, 3)
            truth = np.stack([workload.radiance(xs, np.full(len(xs), l)).reshape(H, W, 3) for l in range(L)])
            m = np.repeat(hit[None], L, 0)
            e = np.abs(img[m] - truth[m]).sum() / max(np.abs(truth[m]).sum(), 1e-30)
            errs.append((fr, float(e)))
            bad = bad or not np.isfinite(img).all() or st.nonfinite_grads > 0
    torch.cuda.synchronize()
    P = np.concatenate([cache.params_rows(l) for l in range(L)])
    e1 = [e for fr, e in errs if frames - 64 <= fr < frames]
    e2 = [e for fr, e in errs if fr >= 2 * frames - 64]
    return {"variant": name, "hparams": over, "path": "screen",
            "rel_error_moving_last64": float(np.mean(e1)), "rel_error_still_last64": float(np.mean(e2)),
            "max_extent_es": float(np.exp(P[:, 10:13]).max()), "max_abs_colour": float(np.abs(P[:, 7:10]).max()),
            "nonfinite": bool(bad or not np.isfinite(P).all()), "curve": errs}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--frames", type=int, default=256)
    ap.add_argument("--firefly", type=float, default=0.0)
    ap.add_argument("--screen", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    out = {"protocol": "viewport half-space turning once about z over `frames` frames, then still "
                       "for `frames`; held-out lookups over the visible half vs the synthetic truth",
           "config": workload.CONFIGS[args.config]["name"], "frames_per_phase": args.frames,
           "firefly": args.firefly,
           "results": []}
    for n, o in VARIANTS.items():
        try:
            if args.screen:
                out["results"].append(run_screen(args.config, args.frames, n, o, dev))
            else:
                out["results"].append(run(args.config, args.frames, n, o, dev, args.firefly))
        except Exception as e:           # e.g. exploding Gaussians overflow the culling lists
            out["results"].append({"variant": n, "hparams": o, "failed": str(e)[:300]})
        torch.cuda.synchronize()
    print(json.dumps(out))


if __name__ == "__main__":
    main()

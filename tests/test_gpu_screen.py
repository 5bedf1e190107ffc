"""Screen-space cache images (next row f1, sec.3.1 / P:189 sec.3.5 / P:375) through the
C ABI (-m gpu) against the fp64 screen-space oracle (oracle/screen_oracle.c, pinned in
tests/test_screen_oracle_pins.py).

Bars: forward |dy| <= 1e-5 |y| + 1e-6 max|y| per pixel and channel, except the pixels the
oracle marks ambiguous (a discrete decision within 1e-4 of its threshold, reading A23),
counted; gradients (the derivative of the oracle's forward, by fp64 central differences) under
both bars of SURVEY 8(c) per (level, group); Adam loss curve within 1 %."""
import numpy as np
import pytest

import oracle
import workload
from test_gpu_parity import check_grad_group, cuda, rows

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gsc():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2507_19718_b200 as m
    assert torch.cuda.is_available()
    return m


def camera(gsc, W, H, f, dist=3.0, rot=(0.15, -0.2, 0.05)):
    from scipy.spatial.transform import Rotation
    R = Rotation.from_rotvec(rot).as_matrix()
    view = np.hstack([R, np.array([[0.02], [-0.03], [dist]])])
    cam = gsc.make_camera(W, H, f, f * 1.05, W / 2 + 0.3, H / 2 - 0.2, view)
    ocam = dict(width=W, height=H, fx=float(np.float32(f)), fy=float(np.float32(f * 1.05)),
                cx=float(np.float32(W / 2 + 0.3)), cy=float(np.float32(H / 2 - 0.2)),
                view=np.array(cam.view[:], np.float64).reshape(3, 4), znear=float(np.float32(0.2)))
    return cam, ocam


def scene(gsc, counts, seed=3, max_opacity=0.8, hparams=None):
    pos, alb = workload.init_cloud(1)
    pos, alb = pos[:counts[0]], alb[:counts[0]]
    c = gsc.GSCache(counts, cuda(pos), cuda(alb), seed=seed, hparams=hparams)
    r = np.random.default_rng(seed)
    for l in range(len(counts)):
        Pl = c.params_rows(l)
        Pl[:, 3:7] = r.normal(size=(len(Pl), 4)).astype(np.float32)
        Pl[:, 10:13] += r.uniform(0.5, 1.5, (len(Pl), 3)).astype(np.float32)     # visible splats
        w = r.uniform(0.2, max_opacity, len(Pl))
        Pl[:, 13] = np.log(w / (1 - w)).astype(np.float32)
        c.set_params_rows(l, Pl)
    return c


def check_image(y, yo, amb, what, max_amb=1e-3, rel=1e-5):
    y, yo = np.asarray(y, np.float64), np.asarray(yo, np.float64)
    tol = rel * np.abs(yo) + 1e-6 * max(np.abs(yo).max(), 1e-30)
    bad = (np.abs(y - yo) > tol).any(axis=-1)
    assert not np.any(bad & (amb == 0)), (what, np.argwhere(bad & (amb == 0))[:5],
                                          np.abs(y - yo)[bad & (amb == 0)][:5])
    assert (bad & (amb != 0)).sum() <= max(5, max_amb * bad.size), (what, (bad & (amb != 0)).sum())


def test_render_matches_oracle(gsc):
    """All levels of a rotated, anisotropic 3-level cache, 200 x 150 pixels, one joint raster."""
    c = scene(gsc, [1500, 400, 100])
    cam, ocam = camera(gsc, 200, 150, 180.0)
    img, T = c.render(cam, with_T=True)
    img, T = img.cpu().numpy(), T.cpu().numpy()
    P = rows(c)
    for l in range(3):
        yo, To, amb = oracle.render(P[c.goff[l]:c.goff[l + 1]], ocam)
        assert (yo > 0).mean() > 0.2
        check_image(img[l], yo, amb, f"level {l}")
        okT = amb == 0
        np.testing.assert_allclose(T[l][okT], To[okT], rtol=1e-5, atol=1e-6)
    one = c.render(cam, level=1).cpu().numpy()                        # a single level alone
    np.testing.assert_array_equal(one[0], img[1])


def test_render_full_hd_sampled(gsc):
    """configs[2]'s 87,040-Gaussian cache at 1920 x 1080, every level, 3000 sampled pixels
    against the oracle computed pixel by pixel."""
    pos, alb = workload.init_cloud(2)
    c = gsc.GSCache(workload.CONFIGS[2]["counts"], cuda(pos), cuda(alb), seed=2)
    cam, ocam = camera(gsc, 1920, 1080, 1400.0)
    img = c.render(cam).cpu().numpy()
    P = rows(c)
    r = np.random.default_rng(4)
    pix = r.choice(1920 * 1080, 3000, replace=False)
    for l in range(4):
        yo, _, amb = oracle.render(P[c.goff[l]:c.goff[l + 1]], ocam, pix=pix)
        y = img[l].reshape(-1, 3)[pix]
        check_image(y, yo.reshape(-1, 3)[pix], amb.reshape(-1)[pix], f"full HD level {l}")
        assert (yo.reshape(-1, 3)[pix] > 0).mean() > 0.05


def _tiny(gsc, seed=5, hparams=None):
    c = scene(gsc, [24, 8], seed=seed, max_opacity=0.7, hparams=hparams)
    cam, ocam = camera(gsc, 48, 40, 40.0)
    P = rows(c)
    r = np.random.default_rng(seed)
    imgs = np.stack([oracle.render(P[c.goff[l]:c.goff[l + 1]], ocam)[0] for l in range(2)])
    target = imgs * r.uniform(0.3, 2.0, imgs.shape) + r.uniform(0, 0.05, imgs.shape)
    valid = (r.random((2, 40, 48)) < 0.85).astype(np.uint8)
    return c, cam, ocam, P, target, valid


def test_fit_image_gradients_match_finite_differences(gsc):
    """The screen-space backward (compositing + EWA + projection chain rule) against fp64
    central finite differences of the oracle's Eq. 4 image loss (mode 0: frozen denominator),
    all 14 raw parameters, both gradient bars; no pixel of the scene is A23-ambiguous and no
    alpha reaches the 0.99 clamp (opacity <= 0.7), so the loss is smooth at the point."""
    c, cam, ocam, P, target, valid = _tiny(gsc)
    for l in range(2):
        assert not oracle.render(P[c.goff[l]:c.goff[l + 1]], ocam)[2].any()
    c.debug_enable_grads(True)
    st = c.fit_image(cam, cuda(target.astype(np.float32)), cuda(valid))
    torch.cuda.synchronize()
    tot, per = oracle.image_loss(c.goff, P, ocam, target, valid)
    for l in range(2):
        assert st.count[l] == int(valid[l].sum())
        assert abs(st.loss[l] - per[l]) <= 1e-4 * per[l]
    g = np.concatenate([c.debug_grads_rows(l) for l in range(2)]).astype(np.float64)
    go = oracle.image_grad_fd(c.goff, P, ocam, target, valid)
    for l in range(2):
        sl = slice(c.goff[l], c.goff[l + 1])
        for name, cs in oracle.GROUP_SLICES.items():
            check_grad_group(g[sl, cs], go[sl, cs], f"screen level {l} {name}")


def test_fit_image_gradients_full_quotient(gsc):
    """loss_grad_mode 1 (Eq. 4's full quotient as written; reading A10): the gradient
    written by the fused forward raster and back-propagated through the compositing and the
    projection, against fp64 central differences of the oracle's live-denominator image loss."""
    c, cam, ocam, P, target, valid = _tiny(gsc, seed=6, hparams=dict(loss_grad_mode=1))
    c.debug_enable_grads(True)
    c.fit_image(cam, cuda(target.astype(np.float32)), cuda(valid))
    torch.cuda.synchronize()
    g = np.concatenate([c.debug_grads_rows(l) for l in range(2)]).astype(np.float64)
    go = oracle.image_grad_fd(c.goff, P, ocam, target, valid, mode=1)
    for l in range(2):
        sl = slice(c.goff[l], c.goff[l + 1])
        for name, cs in oracle.GROUP_SLICES.items():
            check_grad_group(g[sl, cs], go[sl, cs], f"screen mode 1 level {l} {name}")


def test_fit_image_loss_curve_and_world_consistency(gsc):
    """5 gc_fit_image steps vs the oracle's AdamW on finite-difference gradients (C6 with the
    paper's learning rates and Eq. 5): per-level losses within 1 % at every step; afterwards
    the world-space lookups (records + culling lists rebuilt) match the oracle on the new
    parameters."""
    c, cam, ocam, P, target, valid = _tiny(gsc, seed=9)
    oc = oracle.OracleCache([24, 8], P.copy(), grids=c.grids())
    tg, va = cuda(target.astype(np.float32)), cuda(valid)
    for step in range(5):
        st = c.fit_image(cam, tg, va)
        torch.cuda.synchronize()
        _, per = oracle.image_loss(c.goff, oc.P, ocam, target, valid)
        np.testing.assert_allclose(list(st.loss[:2]), per, rtol=1e-2)
        g = oracle.image_grad_fd(c.goff, oc.P, ocam, target, valid)
        oc.step_with_grad(g)
    x, ln = workload.query_batch(1, S=4000, frame=3)
    ln = np.minimum(ln, 2).astype(np.int32)
    P1 = rows(c)
    y = c.query(cuda(x), cuda(ln)).cpu().numpy()
    yo, lv, _ = oracle.query(c.goff, P1, x.astype(np.float64), ln, grids=c.grids())
    from test_gpu_parity import check_forward
    check_forward(y, yo, P1, c.goff, x, lv, what="world lookups after screen fit")
    # the culling lists the image steps left stale are rebuilt for the new parameters (C8,
    # bit-exact), also when the first reader is gc_debug_cull
    c.fit_image(cam, tg, va)
    torch.cuda.synchronize()
    P2 = rows(c)
    for l in range(2):
        off_o, idx_o = oracle.csr_for(P2[c.goff[l]:c.goff[l + 1]], 3.0, c.grid(l))
        off_g, idx_g = c.debug_cull(l)
        np.testing.assert_array_equal(off_g.astype(np.int64), off_o)
        np.testing.assert_array_equal(idx_g, idx_o)


def test_render_crowded_tiles_capacity_growth(gsc):
    """The sort paths of the render: 10,000 of 12,000 Gaussians clustered into one tile at the
    far camera (> 8192 keys in a tile: the global-sort fallback), spread over tiles of
    257..8192 keys at the near camera (the shared-memory tile sort), opacities from 0.001
    (< 1/255: culled by the opacity-aware bounds) to 0.999 (clamped alpha); the near camera
    needs more keys than the far one (the grow-and-rerun path), and the far camera rendered
    again reproduces its first image bit for bit.  Bar: a pixel of the cluster composites up
    to ~500 layers (T falls to the 1e-4 stop through factors 1 - alpha with alpha <= 0.05), and
    each layer's fp32 product T (1 - alpha) and accumulation c alpha T round once: the forward
    error grows like n u (u = 2^-24), 500 u = 3e-5 relative, so this test uses 1e-4 instead of
    the 1e-5 of shallow stacks (A23)."""
    r = np.random.default_rng(21)
    pos = np.concatenate([r.normal(0, 0.004, (10000, 3)), r.uniform(-0.5, 0.5, (2000, 3))]).astype(np.float32)
    alb = r.uniform(0.1, 1.0, (12000, 3)).astype(np.float32)
    counts = [12000, 300]
    c = gsc.GSCache(counts, cuda(pos), cuda(alb), seed=4)
    for l in range(2):
        Pl = c.params_rows(l)
        Pl[:, 3:7] = r.normal(size=(len(Pl), 4)).astype(np.float32)
        Pl[:, 10:13] = np.log(r.uniform(0.002, 0.02, (len(Pl), 3))).astype(np.float32)
        w = np.concatenate([r.uniform(0.001, 0.003, len(Pl) // 10), r.uniform(0.005, 0.05, len(Pl) - len(Pl) // 10 - 5),
                            np.full(5, 0.999)])
        r.shuffle(w)
        Pl[:, 13] = np.log(w / (1 - w)).astype(np.float32)
        c.set_params_rows(l, Pl)
    P = rows(c)
    far, ofar = camera(gsc, 48, 40, 40.0, dist=6.0)
    near, onear = camera(gsc, 96, 80, 5000.0, dist=3.0)
    first = c.render(far).cpu().numpy()
    img = c.render(near).cpu().numpy()
    again = c.render(far).cpu().numpy()
    np.testing.assert_array_equal(again, first)
    for l in range(2):
        Pl = P[c.goff[l]:c.goff[l + 1]]
        for y, oc, what in ((first[l], ofar, "far"), (img[l], onear, "near")):
            yo, _, amb = oracle.render(Pl, oc)
            assert (yo > 0).mean() > 0.01, what
            check_image(y.reshape(-1, 3), yo.reshape(-1, 3), amb.reshape(-1), f"crowded {what} level {l}",
                        rel=1e-4)


def test_render_degenerate_cameras_and_empty_fit(gsc):
    """Edge cases of the screen path: a camera that sees no Gaussian (no keys: every pixel
    C = 0, T = 1), a 1 x 1 image and a 17 x 9 image (partial tiles) against the oracle, and a
    fit_image step with no valid pixel (k_l = 0 on every level: no optimizer step, parameters
    unchanged, finite statistics)."""
    c = scene(gsc, [300, 60], seed=12)
    P = rows(c)
    away, _ = camera(gsc, 40, 30, 40.0, dist=-3.0)            # the scene behind the camera
    img, T = c.render(away, with_T=True)
    assert np.all(img.cpu().numpy() == 0.0) and np.all(T.cpu().numpy() == 1.0)
    for W, H in ((1, 1), (17, 9)):
        cam, ocam = camera(gsc, W, H, 12.0)
        img = c.render(cam).cpu().numpy()
        for l in range(2):
            yo, _, amb = oracle.render(P[c.goff[l]:c.goff[l + 1]], ocam)
            check_image(img[l].reshape(-1, 3), yo.reshape(-1, 3), amb.reshape(-1), f"{W}x{H} level {l}")
    cam, _ = camera(gsc, 40, 30, 40.0)
    tgt = cuda(np.ones((2, 30, 40, 3), np.float32))
    st = c.fit_image(cam, tgt, cuda(np.zeros((2, 30, 40), np.uint8)))
    torch.cuda.synchronize()
    assert st.count[0] == 0 and st.count[1] == 0 and np.isfinite(st.loss[0]) and st.loss[0] == 0.0
    np.testing.assert_array_equal(rows(c), P)

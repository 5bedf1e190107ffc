"""Pins of the screen-space oracle (next row f1, oracle/screen_oracle.c), -m "not gpu".

The paper rasterizes every cache level with the 3D Gaussian splatting rasterizer (P:68
sec.3.1, after Kerbl et al.): EWA projection, 16x16 tiles, front-to-back alpha compositing.
Each pin checks the oracle against something other than itself: closed forms for a single
Gaussian, a numerically differentiated perspective map (scipy rotations) for the EWA
covariance, the compositing recurrence on hand-built stacks, and Eq. 4 spot values."""
import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import oracle

pytestmark = pytest.mark.filterwarnings("ignore")


def cam(W=64, H=48, f=60.0, view=None):
    v = np.hstack([np.eye(3), np.zeros((3, 1))]) if view is None else view
    return dict(width=W, height=H, fx=f, fy=f * 1.1, cx=W / 2, cy=H / 2, view=v, znear=0.2)


def row(mu, q=(1, 0, 0, 0), c=(1, 1, 1), s=(np.log(0.05),) * 3, w=0.5):
    o = np.log(w / (1 - w))
    return np.array([*mu, *q, *c, *s, o], np.float64)


def test_single_gaussian_closed_form():
    """Isotropic Gaussian on the optical axis: Sigma2 = (f sigma / z)^2 I + 0.3 I, and every
    pixel of its tile rectangle shows chat * w * exp(-|d|^2 / (2 s2)) (one layer, T = 1)."""
    c = cam()
    z, sig, w = 2.0, 0.05, 0.6
    P = row((0, 0, z), c=(0.3, 0.7, 1.2), s=(np.log(sig),) * 3, w=w)[None]
    rgb, T, amb = oracle.render(P, c)
    pr = oracle.project(P, c)[0]
    s2x, s2y = (c["fx"] * sig / z) ** 2 + 0.3, (c["fy"] * sig / z) ** 2 + 0.3
    np.testing.assert_allclose(pr[4:7], [1 / s2x, 0.0, 1 / s2y], rtol=1e-12)
    assert pr[1] == c["cx"] and pr[2] == c["cy"] and pr[3] == z
    x0, x1, y0, y1 = (int(v) for v in pr[11:15])
    py, px = np.mgrid[0:c["height"], 0:c["width"]]
    dx, dy = c["cx"] - (px + 0.5), c["cy"] - (py + 0.5)
    a = w * np.exp(-0.5 * (dx ** 2 / s2x + dy ** 2 / s2y))
    inside = (px // 16 >= x0) & (px // 16 < x1) & (py // 16 >= y0) & (py // 16 < y1) & (a >= 1 / 255)
    want = np.where(inside[..., None], a[..., None] * np.array([0.3, 0.7, 1.2]), 0.0)
    np.testing.assert_allclose(rgb, want, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(T, np.where(inside, 1 - a, 1.0), rtol=1e-12)
    assert not amb.any() and inside.sum() > 50


def test_ewa_covariance_vs_numeric_jacobian():
    """Sigma2 = J W Sigma W^T J^T + 0.3 I with J the Jacobian of the perspective map
    (x, y, z) -> (fx x/z + cx, fy y/z + cy) at the camera-space mean: J by central finite
    differences, Sigma from scipy's rotation, an arbitrary camera rotation."""
    r = np.random.default_rng(1)
    Rv = Rotation.from_rotvec([0.2, -0.3, 0.1]).as_matrix()
    tv = np.array([0.1, -0.05, 2.5])
    c = cam(view=np.hstack([Rv, tv[:, None]]))
    for _ in range(20):
        mu = r.uniform(-0.3, 0.3, 3)
        q = r.normal(size=4)
        s = np.log(r.uniform(0.01, 0.08, 3))
        P = row(mu, q=q, s=s)[None]
        pr = oracle.project(P, c)[0]
        if pr[0] == 0:
            continue
        t = Rv @ mu + tv
        f = lambda x: np.array([c["fx"] * x[0] / x[2] + c["cx"], c["fy"] * x[1] / x[2] + c["cy"]])  # noqa: E731
        J = np.stack([(f(t + h) - f(t - h)) / 2e-6 for h in np.eye(3) * 1e-6], axis=1)
        Rq = Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix()     # scipy order x,y,z,w
        Sig = Rq @ np.diag(np.exp(2 * s)) @ Rq.T
        S2 = J @ Rv @ Sig @ Rv.T @ J.T + 0.3 * np.eye(2)
        np.testing.assert_allclose(pr[1:3], f(t), rtol=1e-12)
        np.testing.assert_allclose(pr[4:7], [np.linalg.inv(S2)[0, 0], np.linalg.inv(S2)[0, 1],
                                             np.linalg.inv(S2)[1, 1]], rtol=1e-6)


def test_front_to_back_order_is_depth_not_index():
    """Two Gaussians on the same pixel ray: the nearer one composites first whatever its
    index: C = c_f a_f + c_b a_b (1 - a_f)."""
    c = cam()
    back = row((0, 0, 3.0), c=(1, 0, 0), w=0.5)
    front = row((0, 0, 2.0), c=(0, 1, 0), w=0.4)
    rgb, T, _ = oracle.render(np.stack([back, front]), c)
    pj = oracle.project(np.stack([back, front]), c)
    px, py = c["width"] // 2, c["height"] // 2            # pixel centre at (cx + .5, cy + .5)
    a = []
    for g in pj:
        dx, dy = g[1] - (px + 0.5), g[2] - (py + 0.5)
        a.append(g[7] * np.exp(-0.5 * (g[4] * dx * dx + g[6] * dy * dy) - g[5] * dx * dy))
    ab, af = a
    np.testing.assert_allclose(rgb[py, px], [ab * (1 - af), af, 0.0], rtol=1e-12)
    np.testing.assert_allclose(T[py, px], (1 - af) * (1 - ab), rtol=1e-12)


def test_transmittance_stop_and_alpha_floor():
    """A stack of alpha-0.95 layers: T = 0.05, 0.0025, 1.25e-4, then 6.25e-6 < 1e-4 stops before
    the 4th layer (3 layers contribute); a layer with alpha < 1/255 contributes nothing."""
    c = cam(f=400.0)
    stack = np.stack([row((0, 0, 1.0 + 0.1 * k), c=(1, 1, 1), s=(np.log(0.5),) * 3, w=0.95) for k in range(6)])
    faint = row((0, 0, 0.9), c=(5, 5, 5), s=(np.log(0.5),) * 3, w=0.003)
    rgb, T, amb = oracle.render(np.vstack([stack, faint[None]]), c)
    py, px = c["height"] // 2, c["width"] // 2
    pj = oracle.project(stack, c)
    a = [g[7] * np.exp(-0.5 * (g[4] * (g[1] - px - .5) ** 2 + g[6] * (g[2] - py - .5) ** 2)
                       - g[5] * (g[1] - px - .5) * (g[2] - py - .5)) for g in pj]
    Tk, want = 1.0, 0.0
    for k in range(3):
        want += a[k] * Tk
        Tk *= 1 - a[k]
    np.testing.assert_allclose(rgb[py, px], [want] * 3, rtol=1e-12)
    np.testing.assert_allclose(T[py, px], Tk, rtol=1e-12)
    assert Tk * (1 - a[3]) < 1e-4 and not amb[py, px]


def test_image_loss_eq4_values():
    """Eq. 4 per level over valid pixels: zero residual -> 0; a target of 2y with the
    denominator frozen at y gives sum y^2/(y + eps)^2 / (3k)."""
    c = cam(W=32, H=32)
    P = np.stack([row((0.05 * i, -0.04 * i, 2.0), c=(0.5, 1.0, 1.5), w=0.5) for i in range(3)])
    goff = [0, 2, 3]
    imgs = np.stack([oracle.render(P[0:2], c)[0], oracle.render(P[2:3], c)[0]])
    tot, per = oracle.image_loss(goff, P, c, imgs)
    assert tot == 0.0
    valid = np.ones((2, 32, 32), np.uint8)
    valid[:, ::2] = 0
    tot, per = oracle.image_loss(goff, P, c, 2 * imgs, valid=valid, denom=imgs)
    for l in range(2):
        y = imgs[l][valid[l] == 1]
        np.testing.assert_allclose(per[l], np.sum(y ** 2 / (y + 0.01) ** 2) / (3 * y.shape[0]), rtol=1e-12)


def test_fd_gradient_of_colour_matches_closed_form():
    """The finite-difference gradient (the tests' definition of the screen-space backward) on
    the colour of a single Gaussian equals the closed form of Eq. 4 with a frozen denominator:
    dL/dc = sum_px -2 (x - y) alpha / (y + eps)^2 / (3k) for c > 0."""
    c = cam(W=32, H=32)
    P = row((0.02, 0.01, 2.0), c=(0.4, 0.8, 1.1), w=0.7)[None]
    img = oracle.render(P, c)[0]
    r = np.random.default_rng(2)
    tgt = img[None] * r.uniform(0.5, 1.5, img.shape)[None]
    g = oracle.image_grad_fd([0, 1], P, c, tgt)
    alpha = img[..., 0] / 0.4
    k = 32 * 32
    want = [np.sum(-2 * (tgt[0, ..., ch] - img[..., ch]) * alpha / (img[..., ch] + 0.01) ** 2) / (3 * k)
            for ch in range(3)]
    np.testing.assert_allclose(g[0, 7:10], want, rtol=1e-6)


def test_fd_gradient_of_colour_full_quotient_closed_form():
    """mode 1 (Eq. 4's full quotient, reading A10): the finite-difference colour gradient
    of a single Gaussian equals the closed form d/dy (x - y)^2 / (y + eps)^2 = -2 (x - y)(x + eps)
    / (y + eps)^3, chained through y = c alpha, summed over pixels and divided by 3k."""
    c = cam(W=32, H=32)
    P = row((0.02, 0.01, 2.0), c=(0.4, 0.8, 1.1), w=0.7)[None]
    img = oracle.render(P, c)[0]
    r = np.random.default_rng(3)
    tgt = img[None] * r.uniform(0.5, 1.5, img.shape)[None]
    g = oracle.image_grad_fd([0, 1], P, c, tgt, mode=1)
    alpha = img[..., 0] / 0.4
    k = 32 * 32
    want = [np.sum(-2 * (tgt[0, ..., ch] - img[..., ch]) * (tgt[0, ..., ch] + 0.01) * alpha
                   / (img[..., ch] + 0.01) ** 3) / (3 * k) for ch in range(3)]
    np.testing.assert_allclose(g[0, 7:10], want, rtol=1e-6)
    g0 = oracle.image_grad_fd([0, 1], P, c, tgt)              # differs from the frozen mode
    assert np.abs(g0[0, 7:10] - g[0, 7:10]).max() > 1e-3 * np.abs(g[0, 7:10]).max()

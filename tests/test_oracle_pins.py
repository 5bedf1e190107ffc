"""Pins of the fp64 oracle against what the paper and mathematics fix (-m "not gpu").

Each test names the passage it pins (P: = PAPER.md line, S: = SPEC.md line) and uses an
independent check: printed values (tests/golden), closed forms, scipy/torch library
routines, finite differences, brute force.  None of them re-types the oracle's formula.
"""
import math

import numpy as np
import pytest
import torch
from scipy.spatial.transform import Rotation
from scipy.special import gammainc

import oracle
import workload


def rand_params(G, r, aniso=True, color_lo=0.3):
    P = np.zeros((G, 14))
    P[:, 0:3] = r.uniform(-0.5, 0.5, (G, 3))
    q = r.normal(size=(G, 4))
    P[:, 3:7] = q * r.uniform(0.5, 2.0, (G, 1))          # unnormalised on purpose (A6)
    P[:, 7:10] = r.uniform(color_lo, 2.0, (G, 3))
    P[:, 10:13] = np.log(r.uniform(0.15, 0.4, (G, 3))) if aniso else np.log(0.25)
    P[:, 13] = r.uniform(-1.0, 1.0, G)
    return P


def scipy_R(q):
    w, x, y, z = q / np.linalg.norm(q)
    return Rotation.from_quat([x, y, z, w]).as_matrix()


# ---------------------------------------------------------------- C7 create
def test_splitmix64_vectors(golden):
    for k, v in golden["splitmix64_vectors"]["value"].items():
        assert oracle.splitmix64(int(k, 16)) == int(v, 16)


def test_permutation_is_stable_argsort_of_keys():
    perm = oracle.permutation(1000, 42)
    assert sorted(perm.tolist()) == list(range(1000))
    keys = [oracle.splitmix64(42 + int(i)) for i in perm]
    assert all(keys[i] <= keys[i + 1] for i in range(999))


def test_cache_size_29400000_bytes(golden):
    """300K/150K/75K levels, 14 fp32 per splat -> 29,400,000 B."""
    counts = golden["level_counts_paper"]["value"]
    N0 = counts[0]
    r = np.random.default_rng(0)
    pos, rgb = r.uniform(-1, 1, (N0, 3)), r.uniform(0, 1, (N0, 3))
    P = oracle.create(counts, pos, rgb, init_log_scale=np.full((N0, 3), -3.0), seed=7)
    assert P.shape == (sum(counts), golden["floats_per_splat"]["value"]["total"])
    assert P.size * 4 == golden["cache_size_bytes"]["value"]
    table = golden["memory_table_MB"]["value"]
    dims = golden["floats_per_splat"]["value"]
    for comp in ("position", "rotation", "color", "scale"):
        for l, n in enumerate(counts):
            assert round(n * dims[comp] * 4 / 2**20, 2) == table[comp][l]
    # opacity: printed values are truncated, not rounded (1.144 -> 1.14, 0.286 -> 0.28)
    for l, n in enumerate(counts):
        assert math.floor(n * 4 / 2**20 * 100) / 100 == table["opacity"][l]


def test_create_nested_levels_and_init_values():
    """replicated and sub-sampled per level (nested subsets); 3DGS-like init."""
    r = np.random.default_rng(1)
    pos, rgb = r.uniform(-1, 1, (256, 3)), r.uniform(0, 1, (256, 3))
    counts = [256, 64, 16]
    P = oracle.create(counts, pos, rgb, seed=3)
    np.testing.assert_array_equal(P[:256, 0:3], pos)               # level 0 in caller order
    perm = oracle.permutation(256, 3)
    np.testing.assert_array_equal(P[256:320, 0:3], pos[perm[:64]])
    np.testing.assert_array_equal(P[320:336, 0:3], pos[perm[:16]])
    assert set(map(tuple, P[320:336, 0:3])) <= set(map(tuple, P[256:320, 0:3]))
    np.testing.assert_array_equal(P[:, 3:7], np.tile([1.0, 0, 0, 0], (336, 1)))
    np.testing.assert_allclose(1 / (1 + np.exp(-P[:, 13])), 0.1, rtol=1e-14)
    np.testing.assert_array_equal(P[256:320, 7:10], rgb[perm[:64]])
    assert np.all(P[:, 10] == P[:, 11]) and np.all(P[:, 11] == P[:, 12])  # isotropic


def test_eq2_unit_grid(golden):
    """regular unit grid -> every point's 3-NN mean is 1, sigma 0 -> s = 0.5."""
    g = np.arange(5.0)
    pts = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    dbar = oracle.knn3_mean(pts)
    np.testing.assert_array_equal(dbar, 1.0)
    s = oracle.eq2_from_dbar(dbar, oracle.diag(pts))
    np.testing.assert_array_equal(s, golden["eq2_examples"]["value"]["unit_grid_s"])


def test_eq2_outlier_cap(golden):
    """mu_N = 1, sigma_N = 1, raw = 10 -> cap 3 -> s = 1.5 (z-score cap)."""
    ex = golden["eq2_examples"]["value"]["outlier"]
    dbar = np.array([10.0] + [8.0 / 9.0] * 81)          # mean 1, population std 1
    assert abs(dbar.mean() - ex["mu"]) < 1e-12 and abs(dbar.std() - ex["sigma"]) < 1e-12
    s = oracle.eq2_from_dbar(dbar, 100.0)
    assert abs(s[0] - ex["s"]) < 1e-12
    np.testing.assert_allclose(s[1:], 4.0 / 9.0, rtol=1e-14)


def test_eq2_duplicate_floor():
    """coincident points -> floored scale (1e-6 * diag), never zero/negative log."""
    r = np.random.default_rng(2)
    pts = np.concatenate([np.zeros((4, 3)), r.uniform(-1, 1, (60, 3))])
    dbar = oracle.knn3_mean(pts)
    assert np.all(dbar[:4] == 0.0)
    d = oracle.diag(pts)
    s = oracle.eq2_from_dbar(dbar, d)
    np.testing.assert_allclose(s[:4], 0.5e-6 * d, rtol=1e-14)


def test_knn_brute_matches_scipy():
    from scipy.spatial import cKDTree
    r = np.random.default_rng(3)
    pts = r.uniform(-1, 1, (500, 3))
    d, _ = cKDTree(pts).query(pts, k=4)
    np.testing.assert_allclose(oracle.knn3_mean(pts), d[:, 1:].mean(1), rtol=1e-13)


def test_diag_matches_numpy():
    """The Eq. 2 floor reference (reading A7: AABB diagonal of the level's points), checked
    against numpy's own min/max/norm rather than against orc_diag."""
    r = np.random.default_rng(11)
    for n in (1, 2, 7, 300):
        pts = r.normal(size=(n, 3)) * r.uniform(0.1, 3.0, 3) + r.uniform(-5, 5, 3)
        want = float(np.linalg.norm(pts.max(0) - pts.min(0)))
        assert abs(oracle.diag(pts) - want) <= 1e-14 * max(want, 1.0)
    assert oracle.diag(np.zeros((5, 3))) == 0.0


def _splitmix64_py(x):
    """SplitMix64 in Python integers; its constants are pinned by the published test vectors
    (test_splitmix64_vectors), independently of the C oracle."""
    m = (1 << 64) - 1
    z = (x + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


@pytest.mark.parametrize("seed", [5, 6])
def test_create_eq2_per_level_matches_kdtree(seed):
    """Pins orc_create's Eq. 2 composition (sec.3.2; reading A7/A9): level l >= 1 is
    the first counts[l] points of the stable argsort of splitmix64(seed + i) (computed here in
    Python), its scale comes from the 3-NN of exactly that level's own points (scipy cKDTree,
    self excluded), mu_N / sigma_N (ddof 0) over that level only, the floor from that level's
    own AABB diagonal, then ln s on all three axes.  Using level 0's points for every level,
    storing s instead of ln s, or a single axis would each fail here."""
    from scipy.spatial import cKDTree
    r = np.random.default_rng(seed)
    N0 = 900
    # clustered cloud: levels differ strongly in density, so level-0 kNN distances differ
    # from each subset's own by a large factor
    centres = r.uniform(-1, 1, (6, 3))
    pos = centres[r.integers(0, 6, N0)] + r.normal(scale=0.05, size=(N0, 3))
    pos[:5] += r.uniform(2, 4, (5, 3))                       # a few outliers for the z-cap
    rgb = r.uniform(0, 1, (N0, 3))
    counts = [900, 225, 56, 14]
    P = oracle.create(counts, pos, rgb, seed=seed)
    keys = [_splitmix64_py(seed + i) for i in range(N0)]
    perm = sorted(range(N0), key=lambda i: (keys[i], i))
    off = 0
    for l, n in enumerate(counts):
        idx = np.arange(n) if l == 0 else np.array(perm[:n])
        pts = pos[idx]
        d, _ = cKDTree(pts).query(pts, k=4)
        dbar = d[:, 1:].mean(1)
        mu, sd = dbar.mean(), dbar.std()
        dg = float(np.linalg.norm(pts.max(0) - pts.min(0)))
        s = np.maximum(np.minimum(mu + 2.0 * sd, dbar), 1e-6 * dg) * 0.5
        got = P[off:off + n, 10:13]
        np.testing.assert_allclose(got, np.repeat(np.log(s)[:, None], 3, 1), rtol=0, atol=1e-12)
        off += n
    # the per-level subsets really differ in scale: a level-0 kNN would be ~2x smaller
    assert np.mean(P[900:1125, 10]) > np.mean(P[:900, 10]) + 0.3


def test_create_unit_grid_log_scale_closed_form():
    """S:345 composed through create: a unit grid level gets s = 0.5 -> log-scale ln 0.5 on
    all three axes (closed form)."""
    g = np.arange(6.0)
    pts = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    P = oracle.create([len(pts)], pts, np.ones_like(pts), seed=1)
    np.testing.assert_array_equal(P[:, 10:13], math.log(0.5))


@pytest.mark.parametrize("kind", ["single", "coincident"])
def test_create_degenerate_level_is_finite(kind):
    """Reading A20: a level of one point, or of coincident points, has diag = 0 and
    no neighbour distance; the Eq. 2 floor then falls back to 1e-6 world units (applied after
    the cap) so that the log-scale stays finite: ln(0.5e-6)."""
    if kind == "single":
        pts = np.array([[0.3, -0.2, 0.1]])
    else:
        pts = np.tile([[0.3, -0.2, 0.1]], (9, 1))
    P = oracle.create([len(pts)], pts, np.ones_like(pts), seed=2)
    np.testing.assert_allclose(P[:, 10:13], math.log(0.5e-6), rtol=1e-14)


# ------------------------------------------------------- C1/C3 evaluator pins
def test_peak_is_v_at_mean():
    """Unnormalised Gaussian (A2): yhat(mu) = v = sigmoid(o) * max(0, c)."""
    r = np.random.default_rng(4)
    P = rand_params(1, r)
    y, _ = oracle.eval_brute(P, P[:, 0:3])
    w = 1 / (1 + np.exp(-P[0, 13]))
    np.testing.assert_allclose(y[0], w * np.maximum(P[0, 7:10], 0), rtol=1e-14)


def test_value_along_principal_axes_scipy_rotation():
    """G(mu + R diag(e^s) u) = exp(-|u|^2/2), with R from scipy (independent convention pin)."""
    r = np.random.default_rng(5)
    for _ in range(20):
        P = rand_params(1, r)
        P[0, 7:10] = 2.0
        P[0, 13] = 0.0                                      # v = 1
        R = scipy_R(P[0, 3:7])
        u = r.normal(size=(50, 3)) * 0.8
        x = P[0, 0:3] + (R @ (np.exp(P[0, 10:13])[:, None] * u.T)).T
        y, _ = oracle.eval_brute(P, x, tau=np.inf)
        np.testing.assert_allclose(y[:, 0], np.exp(-0.5 * (u ** 2).sum(1)), rtol=1e-12)


def test_activation_matches_scipy_covariance_inverse():
    r = np.random.default_rng(6)
    P = rand_params(10, r)
    for row in P:
        A, v, w = oracle.activate(row)
        R = scipy_R(row[3:7])
        Sigma = R @ np.diag(np.exp(2 * row[10:13])) @ R.T
        np.testing.assert_allclose(A, np.linalg.inv(Sigma), rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("tau,tol", [(np.inf, 1e-8), (3.0, 1e-4)])
def test_integral_closed_form(golden, tau, tol):
    """Integral of one term = (2 pi)^{3/2} e^{sum s} F_chi2_3(tau^2) (10^7-point stratified
    quadrature in the Gaussian's frame; scipy's regularised gamma gives F)."""
    gv = golden["gauss_integral"]["value"]
    assert abs((2 * np.pi) ** 1.5 - gv["two_pi_pow_1p5"]) < 1e-9
    assert abs(gammainc(1.5, 4.5) - gv["chi2_3_cdf_9"]) < 1e-11
    assert abs(oracle.chi2_3_cdf(9.0) - gv["chi2_3_cdf_9"]) < 1e-11
    r = np.random.default_rng(7)
    P = rand_params(1, r)
    P[0, 7:10] = 2.0
    P[0, 13] = 0.0
    R = scipy_R(P[0, 3:7])
    sc = np.exp(P[0, 10:13])
    n = 216
    h = 12.0 / n
    g = -6.0 + (np.arange(n) + 0.5) * h
    U = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    if not np.isinf(tau):                                    # stratified jitter for the
        U = U + r.uniform(-0.5, 0.5, U.shape) * h             # discontinuous cut-off case
    X = P[0, 0:3] + (U * sc) @ R.T
    y, _ = oracle.eval_brute(P, X, tau=tau)
    integral = y[:, 0].sum() * h ** 3 * np.prod(sc)
    F = 1.0 if np.isinf(tau) else gammainc(1.5, tau * tau / 2)
    exact = (2 * np.pi) ** 1.5 * np.prod(sc) * F
    assert abs(integral / exact - 1) < tol


def test_mixture_integral_linear_in_v():
    r = np.random.default_rng(8)
    P = rand_params(3, r)
    x = r.uniform(-1, 1, (200, 3))
    y1, _ = oracle.eval_brute(P, x)
    P2 = P.copy()
    P2[:, 7:10] *= 2.0
    y2, _ = oracle.eval_brute(P2, x)
    np.testing.assert_allclose(y2, 2 * y1, rtol=1e-14)


def test_colour_clamp_and_sigmoid():
    """A4/A5: negative raw colour contributes nothing; v scales with sigmoid(o)."""
    P = np.zeros((1, 14))
    P[0, 3] = 1
    P[0, 7:10] = [-1.0, 0.0, 3.0]
    P[0, 10:13] = np.log(0.2)
    P[0, 13] = np.log(3.0)                                   # sigmoid = 0.75
    y, _ = oracle.eval_brute(P, np.zeros((1, 3)))
    np.testing.assert_allclose(y[0], [0, 0, 2.25], rtol=1e-15)


# ------------------------------------------------------------------ C4 loss pins
def _single(Pv, xh):
    x = np.zeros((1, 3))
    return oracle.loss_grad([0, len(Pv)], Pv, x, [1], np.full((1, 3), xh))


def test_hdr_loss_examples(golden):
    ex = golden["hdr_loss_examples"]["value"]
    far = np.zeros((1, 14)); far[0, 3] = 1; far[0, 0] = 50.0; far[0, 10:13] = -2; far[0, 7:10] = 1
    r0 = _single(far, ex[0]["xhat"])                         # yhat = 0
    assert abs(r0["loss"][0] - ex[0]["loss"]) < 1e-9
    one = np.zeros((1, 14)); one[0, 3] = 1; one[0, 10:13] = -2; one[0, 7:10] = 2.0  # v = 1
    r1 = _single(one, ex[1]["xhat"])
    assert abs(r1["yhat"][0, 0] - 1.0) < 1e-15
    assert abs(r1["loss"][0] - ex[1]["loss"]) < 1e-12
    r2 = _single(one, 1.0)                                   # zero residual
    assert r2["loss"][0] == 0.0 and np.all(r2["grad"] == 0.0)


def test_loss_averages_over_3k_valid_samples():
    """P:213 'average the loss over all pixels k' -> per level, valid samples, 3 channels (A11)."""
    far = np.zeros((1, 14)); far[0, 3] = 1; far[0, 0] = 50.0; far[0, 7:10] = 1
    x = np.zeros((4, 3))
    rgb = np.array([[1, 1, 1], [1, 1, 1], [np.nan, 1, 1], [1, 1, 1.0]])
    r = oracle.loss_grad([0, 1], far, x, [1, 1, 1, 0], rgb)
    assert r["count"][0] == 2                                # NaN rgb and n=0 dropped
    assert abs(r["loss"][0] - 10000.0) < 1e-9


# ------------------------------------------------------------- C5 gradient pins
def _tiny_problem(seed, L=2, G=(5, 3), S=48, aniso=True):
    r = np.random.default_rng(seed)
    P = np.concatenate([rand_params(g, r, aniso=aniso, color_lo=0.4) for g in G[:L]])
    P[:, 0:3] *= 0.4
    goff = np.concatenate([[0], np.cumsum(G[:L])])
    x = r.uniform(-0.35, 0.35, (S, 3))
    ln = r.integers(1, L + 1, S).astype(np.int32)
    rgb = r.uniform(0.0, 3.0, (S, 3))
    return goff, P, x, ln, rgb


def _fd(fun, P, h=1e-6):
    g = np.zeros_like(P)
    for j in range(P.shape[0]):
        for k in range(P.shape[1]):
            Pp, Pm = P.copy(), P.copy()
            Pp[j, k] += h
            Pm[j, k] -= h
            g[j, k] = (fun(Pp) - fun(Pm)) / (2 * h)
    return g


def test_coefficient_gradients_vs_finite_differences():
    """The oracle's coefficient gradients (C5: dL/dmu, dL/dA, dL/dv before the chain rule, the
    quantity gc_debug_coef_grads exposes) against central finite differences of the loss in
    the raw parameters, composed by hand through scipy's rotation: dL/dmu = FD(position);
    dL/dc_ch = w dL/dv_ch (c > 0); dL/ds_k = -2 e^{-2 s_k} (R^T dA R)_kk."""
    goff, P, x, ln, rgb = _tiny_problem(12, L=1, G=(5,), S=40)

    def loss(Pp):
        return oracle.loss_grad(goff, Pp, x, ln, rgb, tau=np.inf, mode=1)["loss"].sum()

    r = oracle.loss_grad(goff, P, x, ln, rgb, tau=np.inf, mode=1)
    cg = r["coef"]
    fd = _fd(loss, P)
    np.testing.assert_allclose(cg[:, 0:3], fd[:, 0:3], rtol=1e-6, atol=1e-9)
    w = 1.0 / (1.0 + np.exp(-P[:, 13]))
    np.testing.assert_allclose(w[:, None] * cg[:, 9:12], fd[:, 7:10], rtol=1e-6, atol=1e-9)
    for j in range(len(P)):
        R = scipy_R(P[j, 3:7])
        a = cg[j]
        dA = np.array([[a[3], a[6], a[7]], [a[6], a[4], a[8]], [a[7], a[8], a[5]]])
        ds = -2.0 * np.exp(-2.0 * P[j, 10:13]) * np.diag(R.T @ dA @ R)
        np.testing.assert_allclose(ds, fd[j, 10:13], rtol=1e-6, atol=1e-9)


def test_grad_allowance_bounds_actual_cutoff_flips():
    """The A3 boundary allowance (oracle.grad_allowance, test infrastructure) must bound what
    flipping the ambiguous pairs really does: the gradients with the cut-off moved to
    tau^2 (1 -+ 0.9e-4) differ from the tau^2 ones by at most the allowance (amb_rel 1e-4)."""
    r = np.random.default_rng(40)
    G = 60
    P = rand_params(G, r)
    P[:, 0:3] *= 0.8
    x = r.uniform(-0.6, 0.6, (20000, 3))
    ln = np.ones(len(x), np.int32)
    rgb = r.uniform(0, 2, (len(x), 3))
    goff = [0, G]
    base = oracle.loss_grad(goff, P, x, ln, rgb, tau=3.0)
    al = oracle.grad_allowance(goff, P, x, ln, rgb, tau=3.0)
    assert al["n_amb"] > 0
    for f in (1 - 0.9e-4, 1 + 0.9e-4):
        t = 3.0 * math.sqrt(f)
        o = oracle.loss_grad(goff, P, x, ln, rgb, tau=t)
        for key, a in (("grad", al["raw"]), ("coef", al["coef"])):
            d = np.abs(o[key] - base[key])
            assert np.all(d <= a * 1.01 + 1e-15), (key, f, (d - a).max())
        assert np.abs(o["grad"] - base["grad"]).max() > 0      # some pair really flipped


def test_grad_condition_magnitudes():
    """Reading A21's kappa (oracle.grad_allowance(cond=True)): never below |grad| (raw and
    coefficient layouts), and equal to it where every summed term has one sign -- with all
    targets 0 every loss gradient g_i is positive (C5, mode 0: -2(0 - y)/(y+eps)^2 > 0), so the
    colour-amplitude coefficient gradient sum_i g_i e_ij has no cancellation."""
    r = np.random.default_rng(41)
    G = 40
    P = rand_params(G, r)
    P[:, 0:3] *= 0.8
    x = r.uniform(-0.6, 0.6, (5000, 3))
    ln = np.ones(len(x), np.int32)
    goff = [0, G]
    for rgb, same_sign in ((r.uniform(0, 2, (len(x), 3)), False), (np.zeros((len(x), 3)), True)):
        base = oracle.loss_grad(goff, P, x, ln, rgb, tau=3.0)
        kap = oracle.grad_allowance(goff, P, x, ln, rgb, tau=3.0, cond=True)
        for key in ("grad", "coef"):
            k = kap["raw" if key == "grad" else key]
            assert np.all(k >= np.abs(base[key]) * (1 - 1e-12) - 1e-300), key
        if same_sign:
            np.testing.assert_allclose(kap["coef"][:, 9:12], np.abs(base["coef"][:, 9:12]), rtol=1e-12)
        else:
            assert np.any(kap["coef"][:, 0:3] > 1.5 * np.abs(base["coef"][:, 0:3]))


def _check_groups(g, fd, tol):
    for name, sl in oracle.GROUP_SLICES.items():
        a, b = g[:, sl], fd[:, sl]
        assert np.linalg.norm(b) > 1e-8, name
        rel = np.linalg.norm(a - b) / np.linalg.norm(b)
        assert rel < tol, (name, rel)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_gradients_full_quotient_vs_finite_differences(seed):
    """mode 1: analytic raw gradients of sum_l L_l vs central FD, all 5 groups."""
    goff, P, x, ln, rgb = _tiny_problem(seed)
    tau = np.inf
    res = oracle.loss_grad(goff, P, x, ln, rgb, tau=tau, mode=1)
    fd = _fd(lambda Q: oracle.loss_grad(goff, Q, x, ln, rgb, tau=tau, mode=1)["loss"].sum(), P)
    _check_groups(res["grad"], fd, 1e-6)


@pytest.mark.parametrize("seed", [3, 4])
def test_gradients_stopgrad_vs_fd_of_frozen_surrogate(seed):
    """mode 0 (reading A10): gradient of sum (xhat - yhat)^2/(yhat0 + eps)^2/(3k) with the
    denominator frozen at the current yhat0 -- FD of that surrogate via oracle.query."""
    goff, P, x, ln, rgb = _tiny_problem(seed)
    tau = np.inf
    res = oracle.loss_grad(goff, P, x, ln, rgb, tau=tau, mode=0)
    y0, lv, _ = oracle.query(goff, P, x, ln, tau=tau)
    k = np.bincount(lv, minlength=len(goff) - 1)[lv]

    def sur(Q):
        y, _, _ = oracle.query(goff, Q, x, ln, tau=tau)
        return (((rgb - y) ** 2 / (y0 + 0.01) ** 2).sum(1) / (3 * k)).sum()

    _check_groups(res["grad"], _fd(sur, P), 1e-6)


def test_gradients_with_cutoff_are_pairwise_restricted():
    """With tau = 3, FD agrees away from the indicator boundary (no gradient through it)."""
    goff, P, x, ln, rgb = _tiny_problem(5)
    res = oracle.loss_grad(goff, P, x, ln, rgb, tau=3.0, mode=1)
    Qm = oracle.q_matrix(P, x)
    assert np.min(np.abs(Qm - 9.0)) > 1e-3                  # no pair near the boundary
    fd = _fd(lambda Q: oracle.loss_grad(goff, Q, x, ln, rgb, tau=3.0, mode=1)["loss"].sum(), P, 1e-7)
    _check_groups(res["grad"], fd, 1e-5)


def test_isotropic_rotation_gradient_is_zero():
    goff, P, x, ln, rgb = _tiny_problem(6, aniso=False)
    res = oracle.loss_grad(goff, P, x, ln, rgb, tau=np.inf, mode=1)
    scale = np.abs(res["grad"]).max()
    assert np.abs(res["grad"][:, 3:7]).max() < 1e-12 * scale


# ------------------------------------------------------------ C6 optimizer pins
def test_adamw_first_step(golden):
    ex = golden["adamw_first_step"]["value"]
    p, m, v = np.array([ex["p0"]]), np.zeros(1), np.zeros(1)
    oracle.adamw(p, m, v, np.array([ex["grad"]]), ex["lr"], ex["wd"], 0.9, 0.999, 1e-8, 1)
    assert abs(p[0] - ex["p1"]) < 1e-12


def test_adamw_zero_grad_decay_and_nonfinite_skip():
    p, m, v = np.array([2.0, 3.0]), np.zeros(2), np.zeros(2)
    bad = oracle.adamw(p, m, v, np.array([0.0, np.nan]), 0.1, 0.01, 0.9, 0.999, 1e-8, 1)
    assert bad == 1
    assert abs(p[0] - 2.0 * (1 - 0.1 * 0.01)) < 1e-15 and p[1] == 3.0 and m[1] == 0 and v[1] == 0


def test_adamw_matches_torch_adamw():
    """Library routine pin: torch.optim.AdamW (fp64, CPU) over 20 steps, lambda>0 and =0."""
    r = np.random.default_rng(9)
    for wd in (1e-2, 0.0):
        p0 = r.normal(size=50)
        grads = r.normal(size=(20, 50))
        p, m, v = p0.copy(), np.zeros(50), np.zeros(50)
        tp = torch.tensor(p0.copy(), dtype=torch.float64, requires_grad=True)
        opt = torch.optim.AdamW([tp], lr=0.05, betas=(0.9, 0.999), eps=1e-8, weight_decay=wd)
        for s in range(20):
            oracle.adamw(p, m, v, grads[s], 0.05, wd, 0.9, 0.999, 1e-8, s + 1)
            tp.grad = torch.tensor(grads[s])
            opt.step()
        np.testing.assert_allclose(p, tp.detach().numpy(), rtol=1e-12, atol=1e-14)


def test_zero_lr_group_is_frozen():
    """Reading A16 (P:267 scale LR 0; P:430 covariance optimization "by default ... disabled"):
    with the default hyper-parameters the scale group's parameters AND moments never move,
    while the other groups step; with scale LR > 0 (the -CO variant) they do move."""
    r = np.random.default_rng(21)
    G = 6
    P = rand_params(G, r)
    x = r.uniform(-0.6, 0.6, (200, 3))
    ln = np.ones(200, np.int32)
    rgb = r.uniform(0, 2, (200, 3))
    oc = oracle.OracleCache([G], P, hp=dict(tau=np.inf))
    for _ in range(3):
        oc.fit(x, ln, rgb)
    np.testing.assert_array_equal(oc.P[:, 10:13], P[:, 10:13])
    assert np.all(oc.M[:, 10:13] == 0) and np.all(oc.V[:, 10:13] == 0)
    assert np.all(oc.M[:, 0:3] != 0) and np.any(oc.P[:, 0:3] != P[:, 0:3])
    oc2 = oracle.OracleCache([G], P, hp=dict(tau=np.inf, lr=[1.16e-3, 1e-3, 1.25e-2, 1.25e-2, 0.15]))
    oc2.fit(x, ln, rgb)
    assert np.all(oc2.P[:, 10:13] != P[:, 10:13]) and np.all(oc2.V[:, 10:13] > 0)


def test_lr_schedule_eq5(golden):
    for ex in golden["lr_schedule_examples"]["value"]:
        t = math.e if ex["t"] == "e" else ex["t"]
        if ex["t"] == "e":
            assert abs(1.0 / (1.0 + math.log(t)) - ex["ratio"]) < 1e-15
        else:
            assert abs(oracle.lr_schedule(1.0, t) - ex["ratio"]) < 1e-6


def test_fit_step_uses_schedule_and_skips_empty_levels():
    goff, P, x, ln, rgb = _tiny_problem(10)
    ln[:] = 1                                                 # only level 0 has samples
    c = oracle.OracleCache([5, 3], P, hp=dict(lr=[1e-2] * 5))
    r1 = c.fit(x, ln, rgb)
    assert r1["stepped"] and r1["t"] == 1 and list(c.adam_step) == [1, 0]
    np.testing.assert_array_equal(c.P[5:], P[5:])             # level 1 untouched (A12)
    assert np.any(c.P[:5] != P[:5])
    r2 = c.fit(x, np.zeros_like(ln), rgb)                     # no valid sample: no-op
    assert not r2["stepped"] and c.t.value == 1
    # first step moves each non-zero-gradient element by ~lr (Adam, bias-corrected)
    c2 = oracle.OracleCache([5, 3], P, hp=dict(lr=[1e-2] * 5, weight_decay=[0] * 5))
    g = c2.fit(x, ln, rgb)["grad"]
    d = c2.P[:5] - P[:5]
    mask = np.abs(g[:5]) > 1e-3
    np.testing.assert_allclose(d[mask], -1e-2 * np.sign(g[:5][mask]), rtol=1e-4)


# ------------------------------------------------------------- C2 level pins
def test_level_assignment_bruteforce():
    L = 4
    ln = np.array([-3, -1, 0, 1, 2, 3, 4, 5, 9, 1000], np.int32)
    want = [-1, -1, -1, 0, 1, 2, 3, 3, 3, 3]
    x = np.zeros((len(ln), 3))
    assert oracle.level_of(ln, L, x).tolist() == want
    x[3, 1] = np.inf
    assert oracle.level_of(ln, L, x)[3] == -1


# ------------------------------------------------------------ C8 culling pins
def _grid_for(P, cells):
    lo = P[:, 0:3].min(0) - 0.3
    hi = P[:, 0:3].max(0) + 0.3
    dims = np.array(cells, np.int32)
    return lo, dims / (hi - lo), dims


@pytest.mark.parametrize("cells", [(7, 5, 6), (1, 1, 1), (20, 20, 20)])
def test_culling_contains_every_supported_pair(cells):
    r = np.random.default_rng(11)
    P = rand_params(40, r)
    P[:, 10:13] = np.log(r.uniform(0.03, 0.2, (40, 3)))
    origin, inv, dims = _grid_for(P, cells)
    off, idx = oracle.csr_for(P, 3.0, (origin, inv, dims))
    x = np.concatenate([r.uniform(-0.9, 0.9, (3000, 3)),
                        P[:, 0:3] + r.normal(scale=0.1, size=(40, 3))])
    Q = oracle.q_matrix(P, x)
    cell = oracle.sample_cell(x, origin, inv, dims)
    lin = (cell[:, 2] * dims[1] + cell[:, 1]) * dims[0] + cell[:, 0]
    inside = 0
    for i in range(len(x)):
        lst = set(idx[off[lin[i]]:off[lin[i] + 1]].tolist())
        need = np.nonzero(Q[i] <= 9.0 * (1 + 1e-6))[0]
        inside += len(need)
        assert set(need.tolist()) <= lst
    assert inside > 100
    for c in range(len(off) - 1):                           # ascending lists
        seg = idx[off[c]:off[c + 1]]
        assert np.all(np.diff(seg) > 0)


def test_culled_evaluator_equals_brute_force():
    r = np.random.default_rng(12)
    P = np.concatenate([rand_params(60, r), rand_params(20, r)])
    P[:, 10:13] = np.log(r.uniform(0.03, 0.15, (80, 3)))
    goff = [0, 60, 80]
    grids = [_grid_for(P[0:60], (9, 8, 7)), _grid_for(P[60:80], (4, 4, 4))]
    x = r.uniform(-0.7, 0.7, (4000, 3))
    ln = r.integers(0, 4, 4000)
    yb, lvb, npb = oracle.query(goff, P, x, ln)
    yc, lvc, npc = oracle.query(goff, P, x, ln, grids=grids)
    assert npb == npc and npb > 1000
    np.testing.assert_array_equal(lvb, lvc)
    np.testing.assert_allclose(yc, yb, rtol=1e-13, atol=1e-300)
    rgb = r.uniform(0, 2, (4000, 3))
    gb = oracle.loss_grad(goff, P, x, ln, rgb)
    gc = oracle.loss_grad(goff, P, x, ln, rgb, grids=grids)
    np.testing.assert_allclose(gc["loss"], gb["loss"], rtol=1e-12)
    np.testing.assert_allclose(gc["grad"], gb["grad"], rtol=1e-9, atol=1e-14)


def test_cull_bound_is_transcendental_free_and_tight():
    """C8: the exp-free bound U_b exceeds e^{s_b} by a factor in (2^{1/32}, 2^{2/32}]."""
    P = np.zeros((1, 14)); P[0, 3] = 1.0
    n = 2_000_000_000                                        # 1e-7 cells: resolution << h
    inv = n / 200.0
    for s in np.linspace(-6, 1, 57):
        P[0, 10:13] = s
        rng, r2 = oracle.cull_ranges(P, 1.0, np.zeros(3) - 100.0, np.full(3, inv),
                                     np.full(3, n, np.int32))
        h = (rng[0, 3] - rng[0, 0] + 1) / (2 * inv)          # half extent in world units
        ratio = h / np.exp(s)
        assert 2 ** (1 / 32) * (1 - 1e-4) < ratio < 2 ** (2 / 32) * (1 + 1e-4), (s, ratio)
        assert 2 ** (1 / 32) < np.sqrt(r2[0]) / np.exp(s) <= 2 ** (2 / 32)


def test_cull_range_isotropic_ignores_rotation_and_contains_ball():
    """C8 isotropic case: a ball's extent does not depend on the quaternion (h = tau U), and
    every point of the tau e^s ball lies inside the cell range."""
    r = np.random.default_rng(21)
    grid = (np.zeros(3) - 1.0, np.full(3, 37.3), np.full(3, 75, np.int32))
    for _ in range(200):
        P = np.zeros((2, 14))
        P[:, 0:3] = r.uniform(-0.8, 0.8, 3)
        P[:, 10:13] = r.uniform(-4.5, -2.0)
        P[0, 3] = 1.0
        P[1, 3:7] = r.normal(size=4)                          # arbitrary rotation
        rng, r2 = oracle.cull_ranges(P, 3.0, *grid)
        np.testing.assert_array_equal(rng[0], rng[1])
        assert r2[0] == r2[1]
        u = r.normal(size=(500, 3)); u /= np.linalg.norm(u, axis=1, keepdims=True)
        pts = P[0, 0:3] + u * 3.0 * np.exp(P[0, 10])        # the ball's surface
        c = oracle.sample_cell(pts, *grid)
        assert np.all(c >= rng[0, :3]) and np.all(c <= rng[0, 3:])


def test_cell_sphere_test_prunes_aabb_corners():
    """C8 list membership = AABB range AND sphere-box test: strictly fewer entries than the
    AABB alone for an isotropic Gaussian straddling cells, and never losing a covered cell."""
    P = np.zeros((1, 14)); P[0, 3] = 1.0; P[0, 10:13] = np.log(0.1)
    P[0, 0:3] = [0.5, 0.5, 0.5]                             # at a cell corner
    grid = (np.zeros(3) - 1.0, np.full(3, 10.0), np.full(3, 20, np.int32))   # edge 0.1
    rng, r2 = oracle.cull_ranges(P, 3.0, *grid)
    aabb = np.prod(rng[0, 3:] - rng[0, :3] + 1)
    off, idx = oracle.build_csr(P, rng, r2, *grid)
    assert 0 < len(idx) < aabb
    # every cell containing a point of the tau-sphere is listed
    r = np.random.default_rng(13)
    u = r.normal(size=(20000, 3)); u /= np.linalg.norm(u, axis=1, keepdims=True)
    pts = P[0, 0:3] + u * 0.3 * r.uniform(0, 1, (20000, 1)) ** (1 / 3)
    c = oracle.sample_cell(pts, *grid)
    lin = (c[:, 2] * 20 + c[:, 1]) * 20 + c[:, 0]
    listed = {cell for cell in range(8000) if off[cell + 1] > off[cell]}
    assert set(lin.tolist()) <= listed


# ----------------------------------------------------- whole-fit pins (oracle)
def test_recovers_known_mixture_from_clean_samples():
    """cfg0 (BASELINE configs[0]): truth = init lattice with means perturbed <= 0.25 sigma
    and random colours; clean targets.  Loss -> <= 1e-3 x initial in 100 steps and
    held-out relative error <= 1e-2 after 300 (schedule off, paper LRs)."""
    pos, rgb, ls = workload.cfg0_lattice()
    P0 = oracle.create([64], pos.astype(np.float64), rgb.astype(np.float64), ls.astype(np.float64), seed=1)
    dmu, col = workload.cfg0_truth_perturbation()
    T = P0.copy()
    T[:, 0:3] += dmu
    T[:, 7:10] = col
    x, ln = workload.cfg0_samples()
    x = x.astype(np.float64)
    y, _ = oracle.eval_brute(T, x)
    c = oracle.OracleCache([64], P0, hp=dict(lr_schedule=0))
    l0 = None
    for s in range(300):
        r = c.fit(x, ln, y)
        l0 = r["loss"].sum() if l0 is None else l0
        if s == 99:
            assert r["loss"].sum() <= 1e-3 * l0
    xh, _ = workload.cfg0_samples(2048, seed=77)
    yt, _ = oracle.eval_brute(T, xh.astype(np.float64))
    yq, _, _ = c.query(xh.astype(np.float64), np.ones(2048, np.int32))
    assert np.abs(yq - yt).sum() / np.abs(yt).sum() <= 1e-2


@pytest.mark.parametrize("mode", [0, 1])
def test_noise2noise_fixed_point(mode):
    """training on noisy targets with E[xhat] = L.  Mode 0 converges to E[xhat];
    mode 1 (full quotient) to (E[xhat^2] + eps E[xhat])/(E[xhat] + eps) (reading A10)."""
    r = np.random.Generator(np.random.Philox(key=5))
    Lt = np.array([1.0, 0.5, 2.0])
    S = 4096
    Ez2 = math.exp(0.25) / 0.25                              # E[(B Z / p)^2] of the noise model
    target = Lt if mode == 0 else (Ez2 * Lt * Lt + 0.01 * Lt) / (Lt + 0.01)
    P = np.zeros((1, 14)); P[0, 3] = 1; P[0, 7:10] = 2 * target * 0.8
    P[0, 10:13] = np.log(0.1)
    c = oracle.OracleCache([1], P, hp=dict(lr_schedule=1, loss_grad_mode=mode,
                                           lr=[0, 0, 5e-2, 0, 0], weight_decay=[0] * 5))
    x, ln = np.zeros((S, 3)), np.ones(S, np.int32)
    ys = []
    for s in range(1000):
        B = r.random(S) < 0.25
        Z = np.exp(0.5 * r.normal(size=S) - 0.125)
        c.fit(x, ln, Lt[None, :] * (B * Z / 0.25)[:, None])
        if s >= 500:
            ys.append(c.query(x[:1], ln[:1])[0][0])
    ratio = np.mean(ys, 0) / target
    if mode == 0:
        np.testing.assert_allclose(ratio, 1.0, atol=0.01)
    else:
        np.testing.assert_allclose(ratio, 1.0, atol=0.05)
        assert np.all(np.mean(ys, 0) / Lt > 4.0)


def test_query_radiance_epilogue_special_cases():
    """Eq. 3: L_hat = L_n prod(sigma)/beta_{n-1}; beta = 1 and prod(sigma) = 1 reduce
    to the cached value; a cache miss probability beta halves -> radiance doubles; natural
    termination keeps a non-zero unbiased sample and only then."""
    y = np.array([[1.0, 2.0, 3.0], [0.5, 0.0, 4.0], [2.0, 2.0, 2.0]])
    np.testing.assert_array_equal(oracle.query_radiance(y), y)
    np.testing.assert_array_equal(oracle.query_radiance(y, np.ones((3, 3)), np.ones(3)), y)
    np.testing.assert_allclose(oracle.query_radiance(y, beta=np.full(3, 0.5)), 2 * y)
    att = np.array([[0.5, 0.25, 1.0]] * 3)
    np.testing.assert_allclose(oracle.query_radiance(y, att), y * att)
    unb = np.array([[0.0, 0.0, 0.0], [0.0, 1e-3, 0.0], [7.0, 0.0, 0.0]])
    out = oracle.query_radiance(y, att, np.full(3, 0.8), unb)
    np.testing.assert_allclose(out[0], y[0] * att[0] / 0.8)
    np.testing.assert_array_equal(out[1], unb[1])
    np.testing.assert_array_equal(out[2], unb[2])


# ------------------------------------------------------------------ Algorithm 1 (f3)
def test_alg1_hand_cases():
    """Alg. 1 on hand-computed paths: a bright path (Tr >= 0.9) always continues
    with its plain throughput and beta unchanged; a dark one terminates iff q < 1 - Tr, and
    otherwise continues with Tr_out / Tr and beta * Tr (eps = 0 here)."""
    # grey albedos 0.5, 0.5 -> Tr_out = 0.25 (all channels), lum = 0.25 (weights sum to 1)
    sig = [[0.5, 0.5, 0.5], [0.5, 0.5, 0.5]]
    for C_, q, term in ((1.0, 0.74, 1), (1.0, 0.76, 0), (4.0, 0.0, 0)):
        t, tr, b = oracle.alg1(sig, 2, C_, 0.8, q, eps=0.0)
        assert t == term
        if C_ == 4.0:                      # Tr = clamp(1.0) >= 0.9: no roulette at all
            np.testing.assert_allclose(tr, 0.25)
            np.testing.assert_allclose(b, 0.8)
        elif term == 0:                    # continued: 0.25 / 0.25 = 1, beta 0.8 * 0.25
            np.testing.assert_allclose(tr, 1.0, rtol=1e-7)
            np.testing.assert_allclose(b, 0.2, rtol=1e-7)
    # luminance weights: a pure-green path of albedo 0.5 -> Tr = 0.7152 * 0.5
    t, tr, b = oracle.alg1([[0.0, 0.5, 0.0]], 1, 1.0, 1.0, 0.99, eps=0.0)
    assert t == 0 and abs(b - 0.3576) < 1e-6 and abs(tr[1] - 0.5 / 0.3576) < 1e-5
    t, _, _ = oracle.alg1([[0.0, 0.5, 0.0]], 1, 1.0, 1.0, 0.6, eps=0.0)
    assert t == 1                          # q = 0.6 < 1 - 0.3576


def test_alg1_roulette_is_unbiased():
    """Throughput importance sampling is unbiased: over q ~ U(0,1), E[continue *
    Tr_out] = prod sigma (eps = 0), and the cascaded beta is the probability of
    reaching the next vertex, E[1{reached} / beta_{n+1}] = 1 -- integrated exactly over q,
    since the decision is a threshold at q = 1 - Tr."""
    r = np.random.default_rng(3)
    for _ in range(50):
        n = int(r.integers(1, 6))
        sig = r.uniform(0.05, 0.95, (n, 3))
        C_ = float(r.uniform(0.2, 3.0))
        beta = float(r.uniform(0.1, 1.0))
        _, tr0, _ = oracle.alg1(sig, n, C_, beta, 1.0, eps=0.0)      # q = 1: never terminates
        plain = np.prod(sig.astype(np.float32), axis=0)
        _, _, bnext = oracle.alg1(sig, n, C_, beta, 1.0, eps=0.0)
        Tr = bnext / beta                                                # the continue probability
        if Tr >= 0.9 * (1 - 1e-6) and np.allclose(tr0, plain, rtol=1e-6):
            continue                                                     # no roulette at this vertex
        # P(continue) = P(q >= 1 - Tr) = Tr; E[continue * Tr_out] = Tr * plain / Tr = plain
        np.testing.assert_allclose(Tr * tr0, plain, rtol=1e-5)
        np.testing.assert_allclose(Tr * (beta / bnext), 1.0, rtol=1e-6)

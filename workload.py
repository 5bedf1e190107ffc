"""workload -- seeded synthetic inputs shared by the oracle side and the CUDA side.

Holds NONE of the method's arithmetic (no mixture evaluation, loss, gradient or optimizer):
only the synthetic scene that stands in for the paper's volume datasets (P:273-289
Table 1) and renderer (sec.3.7), generated with NumPy's Philox counter-based
generator, seed = 1000 + config index.

Scene ("scientific volume" in [-1,1]^3): 8 thin spherical shells (centres U[-0.6,0.6]^3,
radii U[0.15,0.35], thickness 0.03) plus one slab |z-0.1|<0.02, |x|,|y|<0.8.  A point is a
structure chosen proportionally to its area, a uniform point on it, plus N(0, 0.01^2)
jitter -- the first-collision points of delta tracking on iso-structures (sec.3.2).

Radiance per level (two small lights): L_l(x) = 0.5^l sum_m E_m/(|x-p_m|^2+rho_l^2)
(E scaled so that L is O(0.1-1)),
rho_l = 0.1+0.3 l.  Noisy MC sample: xhat = L B Z / p with B~Bernoulli(p=0.25),
Z = exp(0.5 N - 0.125) shared by the channels, so E[xhat] = L (unbiased).
Path lengths: geometric(0.5) (n=1 w.p. 1/2, ...), 5 % of fit samples carry n=0 (dropped).
"""
from __future__ import annotations

import numpy as np

CONFIGS = {
    0: dict(name="cfg0", counts=[64], S=4096, steps=100),
    1: dict(name="cfg1", counts=[4096, 1024, 256], S=262_144, steps=100),
    2: dict(name="cfg2", counts=[65_536, 16_384, 4_096, 1_024], S=2_073_600, steps=100),
    3: dict(name="cfg3", counts=[65_536, 16_384, 4_096, 1_024], S=2_073_600, steps=200),
    4: dict(name="cfg4", counts=[1_048_576, 262_144, 65_536, 16_384, 4_096, 1_024],
            S=16_777_216, steps=50),
}

# light powers scaled so that attenuated radiance is O(0.1-1), the range the paper's learning
# rates adapt to within tens of frames
LIGHTS = [(np.array([1.5, 1.0, 0.5]), np.array([8.0, 7.0, 6.0]) / 8),
          (np.array([-1.2, 1.4, -0.8]), np.array([2.0, 3.0, 5.0]) / 8)]
# cfg3's mid-run "light / transfer-function change": light 1 moves and brightens x1.5,
# higher-order levels dim x0.7
LIGHTS_CHANGED = [(np.array([-0.5, 1.5, 1.5]), np.array([12.0, 10.5, 9.0]) / 8),
                  (np.array([-1.2, 1.4, -0.8]), np.array([2.0, 3.0, 5.0]) / 8)]


def rng_for(cfg: int, stream: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=1000 + cfg + (stream << 32)))


class Scene:
    """The synthetic volume's iso-structures (fixed per seed)."""

    def __init__(self, seed: int = 1000):
        r = np.random.Generator(np.random.Philox(key=seed))
        self.centres = r.uniform(-0.6, 0.6, size=(8, 3))
        self.radii = r.uniform(0.15, 0.35, size=8)
        self.albedo = r.uniform(0.2, 0.9, size=(9, 3))
        shell_area = 4.0 * np.pi * self.radii ** 2
        slab_area = 2 * (1.6 * 1.6)
        a = np.concatenate([shell_area, [slab_area]])
        self.p = a / a.sum()

    def points(self, n: int, r: np.random.Generator):
        """n structure points and their albedo (float64)."""
        k = r.choice(9, size=n, p=self.p)
        out = np.empty((n, 3))
        sh = k < 8
        m = int(sh.sum())
        d = r.normal(size=(m, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        rad = self.radii[k[sh]] + r.uniform(-0.015, 0.015, size=m)
        out[sh] = self.centres[k[sh]] + d * rad[:, None]
        ns = n - m
        out[~sh, 0] = r.uniform(-0.8, 0.8, ns)
        out[~sh, 1] = r.uniform(-0.8, 0.8, ns)
        out[~sh, 2] = 0.1 + r.uniform(-0.02, 0.02, ns)
        out += r.normal(scale=0.01, size=(n, 3))
        return np.clip(out, -1.0, 1.0), self.albedo[k]


def radiance(x: np.ndarray, level: np.ndarray, changed: bool = False) -> np.ndarray:
    """Synthetic ground-truth attenuated radiance of path-length level `level` at x."""
    rho2 = (0.1 + 0.3 * level.astype(np.float64)) ** 2
    out = np.zeros((len(x), 3))
    for p, E in (LIGHTS_CHANGED if changed else LIGHTS):
        d2 = ((x - p) ** 2).sum(1)
        out += E[None, :] / (d2 + rho2)[:, None]
    out *= (0.5 ** level.astype(np.float64))[:, None]
    if changed:
        out *= np.where(level >= 1, 0.7, 1.0)[:, None]
    return out


def path_lengths(n: int, L: int, r: np.random.Generator, p_zero: float = 0.05) -> np.ndarray:
    ln = r.geometric(0.5, size=n).astype(np.int32)
    ln = np.minimum(ln, L + 2)                         # lengths beyond L land in the last level
    ln[r.random(n) < p_zero] = 0
    return ln


def init_cloud(cfg: int):
    """counts[0] init points (float32 pos, float32 albedo) for configs 1-4."""
    c = CONFIGS[cfg]
    sc = Scene(1000 + cfg)
    pos, alb = sc.points(c["counts"][0], rng_for(cfg, 1))
    return pos.astype(np.float32), alb.astype(np.float32)


def fit_batch(cfg: int, frame: int = 0, S: int | None = None, morton: bool = False,
              light_scale: float = 1.0, changed: bool = False):
    """One frame of noisy renderer samples: pos f32[S][3], len i32[S], rgb f32[S][3]."""
    c = CONFIGS[cfg]
    S = c["S"] if S is None else S
    L = len(c["counts"])
    sc = Scene(1000 + cfg)
    r = rng_for(cfg, 100 + frame)
    pos, _ = sc.points(S, r)
    ln = path_lengths(S, L, r)
    lvl = np.clip(np.minimum(ln, L) - 1, 0, None)
    Lx = radiance(pos, lvl, changed) * light_scale
    B = (r.random(S) < 0.25).astype(np.float64)
    Z = np.exp(0.5 * r.normal(size=S) - 0.125)
    rgb = Lx * (B * Z / 0.25)[:, None]
    if morton:
        order = np.argsort(_morton(pos), kind="stable")
        pos, ln, rgb = pos[order], ln[order], rgb[order]
    return pos.astype(np.float32), ln.astype(np.int32), rgb.astype(np.float32)


def query_batch(cfg: int, frame: int = 0, S: int | None = None, morton: bool = False):
    """Cache lookups of one frame: pos f32[S][3], len i32[S] (all >= 1)."""
    c = CONFIGS[cfg]
    S = c["S"] if S is None else S
    L = len(c["counts"])
    sc = Scene(1000 + cfg)
    r = rng_for(cfg, 50_000 + frame)
    pos, _ = sc.points(S, r)
    ln = path_lengths(S, L, r, p_zero=0.0)
    if morton:
        order = np.argsort(_morton(pos), kind="stable")
        pos, ln = pos[order], ln[order]
    return pos.astype(np.float32), ln.astype(np.int32)


def _morton(x: np.ndarray) -> np.ndarray:
    q = np.clip(((x + 1.0) * 512).astype(np.int64), 0, 1023)
    code = np.zeros(len(x), np.int64)
    for b in range(10):
        for a in range(3):
            code |= ((q[:, a] >> b) & 1) << (3 * b + a)
    return code


def cfg0_lattice(jitter_seed: int = 1000):
    """cfg0 geometry: jittered 4x4x4 lattice in [-0.75,0.75]^3, isotropic s = ln 0.15."""
    r = np.random.Generator(np.random.Philox(key=jitter_seed))
    g = np.linspace(-0.75, 0.75, 4)
    pos = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    pos = pos + r.uniform(-0.05, 0.05, size=pos.shape)
    rgb = r.uniform(0.2, 0.9, size=(64, 3))
    log_scale = np.full((64, 3), np.log(0.15))
    return pos.astype(np.float32), rgb.astype(np.float32), log_scale.astype(np.float32)


def cfg0_truth_perturbation(jitter_seed: int = 1000):
    """Known-mixture truth for cfg0: mean offsets (<= 0.25 sigma per axis) and raw colours."""
    r = np.random.Generator(np.random.Philox(key=jitter_seed + 7))
    dmu = r.uniform(-0.25, 0.25, size=(64, 3)) * 0.15
    color = r.uniform(0.5, 4.0, size=(64, 3))
    return dmu, color


def cfg0_samples(S: int = 4096, seed: int = 1000):
    """cfg0 sample positions (uniform in the lattice's box) and path lengths (all 1)."""
    r = np.random.Generator(np.random.Philox(key=seed + 11))
    pos = r.uniform(-0.9, 0.9, size=(S, 3))
    return pos.astype(np.float32), np.ones(S, np.int32)


def primary_hits(view, W, H, fx, fy, cx, cy, seed=1000):
    """Screen-space samples (next row f1): the first structure each pixel's primary ray meets in
    the synthetic scene -- the 8 shells as infinitely thin spheres, the slab as the plane
    z = 0.1 inside |x|, |y| < 0.8 -- for a pinhole camera with world->camera view [R | t]
    (pixel (px, py) through (px + 0.5, py + 0.5), u = fx x/z + cx).  Returns hit points [H][W][3]
    (NaN where the ray misses) and a hit mask.  Geometry only (no method arithmetic)."""
    sc = Scene(seed)
    V = np.asarray(view, np.float64).reshape(3, 4)
    R, t = V[:, :3], V[:, 3]
    o = -R.T @ t                                               # camera centre in the world
    py, px = np.mgrid[0:H, 0:W]
    dc = np.stack([(px + 0.5 - cx) / fx, (py + 0.5 - cy) / fy, np.ones_like(px, np.float64)], -1)
    d = dc @ R                                                 # R^T dc, per pixel
    d /= np.linalg.norm(d, axis=-1, keepdims=True)
    best = np.full((H, W), np.inf)
    for c, r in zip(sc.centres, sc.radii):
        oc = o - c
        b = d @ oc
        disc = b * b - (oc @ oc - r * r)
        ok = disc >= 0
        sq = np.sqrt(np.where(ok, disc, 0.0))
        for tt in (-b - sq, -b + sq):
            m = ok & (tt > 1e-6) & (tt < best)
            best = np.where(m, tt, best)
    with np.errstate(divide="ignore", invalid="ignore"):
        tz = (0.1 - o[2]) / d[..., 2]
    hz = o + tz[..., None] * d
    m = (tz > 1e-6) & (tz < best) & (np.abs(hz[..., 0]) < 0.8) & (np.abs(hz[..., 1]) < 0.8)
    best = np.where(m, tz, best)
    hit = np.isfinite(best)
    x = np.where(hit[..., None], o + best[..., None] * d, np.nan)
    return x, hit


def screen_targets(x, hit, L, r: np.random.Generator, changed: bool = False):
    """Noisy per-level radiance images of one frame's primary hits: target [L][H][W][3] =
    L_l(x) B Z / p (the fit samples' noise model) and valid [L][H][W] (hit pixels)."""
    H, W = hit.shape
    tgt = np.zeros((L, H, W, 3))
    xs = np.where(hit[..., None], x, 0.0).reshape(-1, 3)
    for l in range(L):
        Lx = radiance(xs, np.full(len(xs), l), changed).reshape(H, W, 3)
        B = (r.random((H, W)) < 0.25).astype(np.float64)
        Z = np.exp(0.5 * r.normal(size=(H, W)) - 0.125)
        tgt[l] = Lx * (B * Z / 0.25)[..., None]
    valid = np.repeat(hit[None], L, 0)
    return np.where(valid[..., None], tgt, 0.0), valid

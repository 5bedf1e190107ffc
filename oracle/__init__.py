"""oracle -- ctypes/numpy wrapper of the plain fp64 CPU oracle (oracle/gscache_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs, never by the product package
``paper_2507_19718_b200``.  It shares no code with the CUDA path.

Every function follows PAPER.md (cited ``P:<line>``) / SURVEY.md section 8(c) (C1-C8);
see the C file's header.  Parameter rows are fp64 ``[G][14]`` in paper order
(P:444-448): position(3), rotation wxyz(4), colour(3), log-scale(3), opacity logit(1).

Parity status: every function here is pinned by tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gscache_oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "screen_oracle.c"), os.path.join(_HERE, "gscache_oracle.h")]
_LIB = os.path.join(_HERE, "liboracle.so")

NP = 14
GROUP_SLICES = {"position": slice(0, 3), "rotation": slice(3, 7), "color": slice(7, 10),
                "scale": slice(10, 13), "opacity": slice(13, 14)}

# Paper defaults (P:267 learning rates; S:472/S:503 AdamW internals; P:210 eps; reading A3 tau)
DEFAULT_HP = dict(lr=[1.16e-3, 1e-3, 1.25e-2, 0.0, 1.5e-1],
                  weight_decay=[0.0, 1e-2, 1e-2, 1e-2, 1e-2],
                  beta1=0.9, beta2=0.999, adam_eps=1e-8, hdr_eps=0.01, tau=3.0,
                  loss_grad_mode=0, lr_schedule=1)


def build(force: bool = False) -> str:
    """Compile the oracle shared library with gcc (-ffp-contract=off, plain -O2)."""
    if force or not os.path.exists(_LIB) or any(os.path.getmtime(_LIB) < os.path.getmtime(f) for f in _SRCS):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                               "-shared", "-o", _LIB, _SRCS[0], _SRCS[1], "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_LIB)
        _lib.orc_splitmix64.restype = C.c_uint64
        _lib.orc_splitmix64.argtypes = [C.c_uint64]
        _lib.orc_diag.restype = C.c_double
        _lib.orc_lr_schedule.restype = C.c_double
        _lib.orc_lr_schedule.argtypes = [C.c_double, C.c_int64]
        _lib.orc_build_csr.restype = C.c_int64
        _lib.orc_adamw.restype = C.c_int64
        _lib.orc_level_of.restype = C.c_int32
    return _lib


def _p(a, dtype):
    """Pointer to a C-contiguous numpy array (None -> NULL)."""
    if a is None:
        return None
    assert a.dtype == dtype and a.flags["C_CONTIGUOUS"], (a.dtype, dtype)
    return a.ctypes.data_as(C.c_void_p)


def _d(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _i64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


# ----------------------------------------------------------------- create (C7)
def splitmix64(x: int) -> int:
    return int(lib().orc_splitmix64(C.c_uint64(x & 0xFFFFFFFFFFFFFFFF)))


def permutation(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, np.int64)
    lib().orc_permutation(C.c_int64(n), C.c_uint64(seed), _p(out, np.int64))
    return out


def knn3_mean(pts) -> np.ndarray:
    pts = _d(pts).reshape(-1, 3)
    out = np.empty(len(pts), np.float64)
    lib().orc_knn3_mean(C.c_int64(len(pts)), _p(pts, np.float64), _p(out, np.float64))
    return out


def diag(pts) -> float:
    pts = _d(pts).reshape(-1, 3)
    return float(lib().orc_diag(C.c_int64(len(pts)), _p(pts, np.float64)))


def eq2_from_dbar(dbar, diag_len: float, zcap: float = 2.0, factor: float = 0.5) -> np.ndarray:
    dbar = _d(dbar)
    out = np.empty_like(dbar)
    lib().orc_eq2_from_dbar(C.c_int64(len(dbar)), _p(dbar, np.float64), C.c_double(diag_len),
                            C.c_double(zcap), C.c_double(factor), _p(out, np.float64))
    return out


def create(counts, init_pos, init_rgb, init_log_scale=None, seed=0, init_opacity=0.1,
           zcap=2.0, factor=0.5) -> np.ndarray:
    counts = _i64(counts)
    pos, rgb = _d(init_pos).reshape(-1, 3), _d(init_rgb).reshape(-1, 3)
    ls = None if init_log_scale is None else _d(init_log_scale).reshape(-1, 3)
    P = np.empty((int(counts.sum()), NP), np.float64)
    lib().orc_create(C.c_int(len(counts)), _p(counts, np.int64), _p(pos, np.float64),
                     _p(rgb, np.float64), _p(ls, np.float64), C.c_uint64(seed),
                     C.c_double(init_opacity), C.c_double(zcap), C.c_double(factor),
                     _p(P, np.float64))
    return P


# ------------------------------------------------------------- activation (C1)
def activate(row):
    row = _d(row)
    A = np.empty(9, np.float64)
    v = np.empty(3, np.float64)
    w = C.c_double()
    lib().orc_activate(_p(row, np.float64), _p(A, np.float64), _p(v, np.float64), C.byref(w))
    return A.reshape(3, 3), v, w.value


# -------------------------------------------------------------- evaluator (C3)
def eval_brute(P, x, tau=3.0, amb_rel=None):
    """yhat [S][3] of ONE level's Gaussians P at points x; optional A3 ambiguity data."""
    P, x = _d(P).reshape(-1, NP), _d(x).reshape(-1, 3)
    y = np.empty((len(x), 3), np.float64)
    npairs = C.c_int64()
    amb = np.empty((len(x), 3), np.float64) if amb_rel is not None else None
    amb_n = np.empty(len(x), np.int32) if amb_rel is not None else None
    lib().orc_eval_brute(C.c_int64(len(P)), _p(P, np.float64), C.c_double(tau), C.c_int64(len(x)),
                         _p(x, np.float64), _p(y, np.float64), C.byref(npairs),
                         C.c_double(amb_rel or 0.0), _p(amb, np.float64), _p(amb_n, np.int32))
    if amb_rel is None:
        return y, npairs.value
    return y, npairs.value, amb, amb_n


def q_matrix(P, x):
    P, x = _d(P).reshape(-1, NP), _d(x).reshape(-1, 3)
    Q = np.empty((len(x), len(P)), np.float64)
    lib().orc_q_matrix(C.c_int64(len(P)), _p(P, np.float64), C.c_int64(len(x)), _p(x, np.float64),
                       _p(Q, np.float64))
    return Q


# ------------------------------------------------------------------ culling (C8)
def sample_cell(x, origin, inv_cell, dims):
    x = _d(x).reshape(-1, 3)
    o, ic, dm = _d(origin), _d(inv_cell), _i32(dims)
    out = np.empty((len(x), 3), np.int32)
    for i in range(len(x)):
        lib().orc_sample_cell(_p(x[i].copy(), np.float64), _p(o, np.float64), _p(ic, np.float64),
                              _p(dm, np.int32), out[i].ctypes.data_as(C.c_void_p))
    return out


def cull_ranges(P, tau, origin, inv_cell, dims):
    """C8: per-Gaussian inclusive cell ranges [G][6] and bounding-sphere radii^2 [G]."""
    P = _d(P).reshape(-1, NP)
    o, ic, dm = _d(origin), _d(inv_cell), _i32(dims)
    rng = np.empty((len(P), 6), np.int32)
    r2 = np.empty(len(P), np.float64)
    lib().orc_cull_ranges(C.c_int64(len(P)), _p(P, np.float64), C.c_double(tau), _p(o, np.float64),
                          _p(ic, np.float64), _p(dm, np.int32), _p(rng, np.int32), _p(r2, np.float64))
    return rng, r2


def build_csr(P, rng, r2, origin, inv_cell, dims):
    """C8 culling lists (cell -> ascending level-local Gaussian indices)."""
    P, rng, r2 = _d(P).reshape(-1, NP), _i32(rng).reshape(-1, 6), _d(r2)
    o, ic, dm = _d(origin), _d(inv_cell), _i32(dims)
    cells = int(dm[0]) * int(dm[1]) * int(dm[2])
    off = np.empty(cells + 1, np.int64)
    args = (C.c_int64(len(rng)), _p(P, np.float64), _p(rng, np.int32), _p(r2, np.float64),
            _p(o, np.float64), _p(ic, np.float64), _p(dm, np.int32), _p(off, np.int64))
    n = lib().orc_build_csr(*args, None)
    idx = np.empty(max(n, 1), np.int32)
    lib().orc_build_csr(*args, _p(idx, np.int32))
    return off, idx[:n]


def csr_for(P, tau, grid):
    """Convenience: the C8 lists of one level for grid = (origin, inv_cell, dims)."""
    o, ic, d = grid
    rng, r2 = cull_ranges(P, tau, o, ic, d)
    return build_csr(P, rng, r2, o, ic, d)


def _grids(grids, L):
    if grids is None:
        return None, None, None
    o = _d([g[0] for g in grids]).reshape(L, 3)
    ic = _d([g[1] for g in grids]).reshape(L, 3)
    dm = _i32([g[2] for g in grids]).reshape(L, 3)
    return o, ic, dm


def query(goff, P, x, length=None, level=-1, tau=3.0, grids=None):
    """Cache lookup (C3) for all levels; grids = [(origin, inv_cell, dims)] -> culled path."""
    goff = _i64(goff)
    L = len(goff) - 1
    P, x = _d(P).reshape(-1, NP), _d(x).reshape(-1, 3)
    S = len(x)
    ln = _i32(length if length is not None else np.zeros(S))
    lv = np.empty(S, np.int32)
    y = np.empty((S, 3), np.float64)
    npairs = C.c_int64()
    o, ic, dm = _grids(grids, L)
    lib().orc_query(C.c_int(L), _p(goff, np.int64), _p(P, np.float64), C.c_double(tau),
                    C.c_int64(S), _p(x, np.float64), _p(ln, np.int32), C.c_int(level),
                    _p(o, np.float64), _p(ic, np.float64), _p(dm, np.int32), _p(lv, np.int32),
                    _p(y, np.float64), C.byref(npairs))
    return y, lv, npairs.value


def query_radiance(yhat, attenuation=None, beta=None, unbiased_rgb=None):
    """Renderer epilogue of a cache hit (next-row f3): natural termination keeps a path's own
    non-zero radiance (sec.3.3.1); otherwise Eq. 3 (sec.3.4.2)
    L_hat = L_n * prod(sigma) / beta_{n-1}.  fp64, elementwise."""
    y = _d(yhat).reshape(-1, 3).copy()
    if attenuation is not None:
        y = y * _d(attenuation).reshape(-1, 3)
    if beta is not None:
        y = y / _d(beta).reshape(-1, 1)
    if unbiased_rgb is not None:
        u = _d(unbiased_rgb).reshape(-1, 3)
        hit = np.any(u != 0.0, axis=1)
        y[hit] = u[hit]
    return y


def alg1(sigma, n, C_, beta, q, eps=1e-6):
    """Algorithm 1 (sec.3.3.2), early path termination, one path, as written:
    Tr_out <- prod_k sigma_k; Tr <- clamp(C lum(Tr_out), 0, 1); if Tr < 0.9: p <- 1 - Tr,
    terminate if q < p, else Tr_out <- Tr_out/(Tr + eps), beta_{n+1} <- beta_n Tr.
    Readings A22: Rec. 709 luminance (0.2126, 0.7152, 0.0722); beta and Tr_out unchanged where
    Alg. 1 assigns nothing.  The decision q < 1 - Tr is taken in fp32 with every operation
    rounded in the written order (the device's precision, so both sides take the same branch);
    returns (terminate, tr_out[3], beta_next) as fp32 values."""
    f = np.float32
    t = [f(1.0), f(1.0), f(1.0)]
    for k in range(int(n)):
        for c in range(3):
            t[c] = f(t[c] * f(sigma[k][c]))
    lum = f(f(f(0.2126) * t[0]) + f(f(0.7152) * t[1]))
    lum = f(lum + f(f(0.0722) * t[2]))
    tr = f(f(C_) * lum)
    tr = f(min(max(tr, f(0.0)), f(1.0)))
    if tr < f(0.9):
        p = f(f(1.0) - tr)
        if f(q) < p:
            return 1, np.array(t, np.float32), f(beta)
        d = f(tr + f(eps))
        return 0, np.array([f(v / d) for v in t], np.float32), f(f(beta) * tr)
    return 0, np.array(t, np.float32), f(beta)


def level_of(length, L, x, rgb=None):
    x = _d(x).reshape(-1, 3)
    rgb = None if rgb is None else _d(rgb).reshape(-1, 3)
    out = np.empty(len(x), np.int32)
    for i in range(len(x)):
        out[i] = lib().orc_level_of(C.c_int32(int(length[i])), C.c_int(L),
                                    _p(x[i].copy(), np.float64),
                                    None if rgb is None else _p(rgb[i].copy(), np.float64))
    return out


# ------------------------------------------------ loss / gradients / optimizer
def loss_grad(goff, P, x, length, rgb, tau=3.0, hdr_eps=0.01, mode=0, grids=None):
    goff = _i64(goff)
    L = len(goff) - 1
    P = _d(P).reshape(-1, NP)
    x, rgb, ln = _d(x).reshape(-1, 3), _d(rgb).reshape(-1, 3), _i32(length)
    S = len(x)
    lv = np.empty(S, np.int32)
    y = np.empty((S, 3), np.float64)
    cnt = np.empty(L, np.int64)
    loss = np.empty(L, np.float64)
    grad = np.empty_like(P)
    cg = np.empty((len(P), 15), np.float64)
    npairs = C.c_int64()
    o, ic, dm = _grids(grids, L)
    lib().orc_loss_grad(C.c_int(L), _p(goff, np.int64), _p(P, np.float64), C.c_double(tau),
                        C.c_double(hdr_eps), C.c_int(mode), C.c_int64(S), _p(x, np.float64),
                        _p(ln, np.int32), _p(rgb, np.float64), _p(o, np.float64),
                        _p(ic, np.float64), _p(dm, np.int32), _p(lv, np.int32), _p(y, np.float64),
                        _p(cnt, np.int64), _p(loss, np.float64), _p(grad, np.float64),
                        C.byref(npairs), _p(cg, np.float64))
    # coefficient gradients in the library's debug layout (gc_debug_coef_grads): dmu (3),
    # dA00 dA11 dA22 dA01 dA02 dA12 (full symmetric elements), dv (3); normalised by 1/(3 k_l)
    coef = np.stack([cg[:, 0], cg[:, 1], cg[:, 2], cg[:, 3], cg[:, 7], cg[:, 11], cg[:, 4],
                     cg[:, 5], cg[:, 8], cg[:, 12], cg[:, 13], cg[:, 14]], axis=1)
    return dict(level=lv, yhat=y, count=cnt, loss=loss, grad=grad, npairs=npairs.value,
                coef=coef)


def grad_allowance(goff, P, x, length, rgb, tau=3.0, hdr_eps=0.01, mode=0, grids=None,
                   amb_rel=1e-4, cond=False):
    """First-order bound of the gradient change that reading A3's fp32 cut-off flips can
    cause (pairs with |Q - tau^2| <= amb_rel tau^2), per Gaussian: coefficient layout like
    loss_grad()['coef'] and raw [G][14]; plus the number of samples with an ambiguous pair.
    cond=True returns instead the condition magnitudes kappa (reading A21): the same gradients
    summed and chained with absolute values, so that a relative perturbation delta of every
    summed term moves a gradient element by at most delta * kappa."""
    goff = _i64(goff)
    L = len(goff) - 1
    P = _d(P).reshape(-1, NP)
    x, rgb, ln = _d(x).reshape(-1, 3), _d(rgb).reshape(-1, 3), _i32(length)
    ac = np.empty((len(P), 15), np.float64)
    ar = np.empty((len(P), NP), np.float64)
    na = C.c_int64()
    o, ic, dm = _grids(grids, L)
    lib().orc_grad_allowance(C.c_int(L), _p(goff, np.int64), _p(P, np.float64), C.c_double(tau),
                             C.c_double(hdr_eps), C.c_int(mode), C.c_int64(len(x)),
                             _p(x, np.float64), _p(ln, np.int32), _p(rgb, np.float64),
                             _p(o, np.float64), _p(ic, np.float64), _p(dm, np.int32),
                             C.c_double(amb_rel), C.c_int(1 if cond else 0), _p(ac, np.float64),
                             _p(ar, np.float64), C.byref(na))
    coef = np.stack([ac[:, 0], ac[:, 1], ac[:, 2], ac[:, 3], ac[:, 7], ac[:, 11], ac[:, 4],
                     ac[:, 5], ac[:, 8], ac[:, 12], ac[:, 13], ac[:, 14]], axis=1)
    return dict(coef=coef, raw=ar, n_amb=na.value)


def adamw(p, m, v, g, lr, wd, beta1, beta2, eps, step):
    """In-place AdamW on fp64 arrays (C6); returns the non-finite count."""
    return int(lib().orc_adamw(C.c_int64(p.size), _p(p, np.float64), _p(m, np.float64),
                               _p(v, np.float64), _p(_d(g), np.float64), C.c_double(lr),
                               C.c_double(wd), C.c_double(beta1), C.c_double(beta2),
                               C.c_double(eps), C.c_int64(step)))


def lr_schedule(eta0: float, t: int) -> float:
    return float(lib().orc_lr_schedule(C.c_double(eta0), C.c_int64(t)))


def hp_vector(hp: dict | None = None, as_float32: bool = True) -> np.ndarray:
    """17-double hyper-parameter vector; as_float32 mirrors the C ABI's float fields."""
    h = dict(DEFAULT_HP)
    if hp:
        h.update(hp)
    f = (lambda v: float(np.float32(v))) if as_float32 else float
    vec = [f(a) for a in h["lr"]] + [f(a) for a in h["weight_decay"]] + [
        f(h["beta1"]), f(h["beta2"]), f(h["adam_eps"]), f(h["hdr_eps"]), f(h["tau"]),
        float(h["loss_grad_mode"]), float(h["lr_schedule"])]
    return np.array(vec, np.float64)


class OracleCache:
    """fp64 oracle of the whole cache state: params, AdamW moments, per-level Adam steps,
    the Eq. 5 schedule counter.  ``fit`` is one gc_fit step (C2-C6)."""

    def __init__(self, counts, P, hp: dict | None = None, grids=None):
        self.counts = _i64(counts)
        self.goff = np.concatenate([[0], np.cumsum(self.counts)]).astype(np.int64)
        self.L = len(self.counts)
        self.P = _d(P).reshape(-1, NP).copy()
        self.M = np.zeros_like(self.P)
        self.V = np.zeros_like(self.P)
        self.adam_step = np.zeros(self.L, np.int64)
        self.t = C.c_int64(0)
        self.hp = hp_vector(hp)
        self.grids = grids

    def reset_schedule(self):
        self.t = C.c_int64(0)

    def fit(self, x, length, rgb):
        x, rgb, ln = _d(x).reshape(-1, 3), _d(rgb).reshape(-1, 3), _i32(length)
        S = len(x)
        cnt = np.empty(self.L, np.int64)
        loss = np.empty(self.L, np.float64)
        grad = np.empty_like(self.P)
        nonfinite = C.c_int64()
        npairs = C.c_int64()
        o, ic, dm = _grids(self.grids, self.L)
        r = lib().orc_fit_step(C.c_int(self.L), _p(self.goff, np.int64), _p(self.P, np.float64),
                               _p(self.M, np.float64), _p(self.V, np.float64),
                               _p(self.adam_step, np.int64), C.byref(self.t),
                               _p(self.hp, np.float64), C.c_int64(S), _p(x, np.float64),
                               _p(ln, np.int32), _p(rgb, np.float64), _p(o, np.float64),
                               _p(ic, np.float64), _p(dm, np.int32), _p(cnt, np.int64),
                               _p(loss, np.float64), _p(grad, np.float64), C.byref(nonfinite),
                               C.byref(npairs))
        return dict(stepped=(r == 0), count=cnt, loss=loss, grad=grad,
                    nonfinite=nonfinite.value, npairs=npairs.value, t=self.t.value)

    def query(self, x, length=None, level=-1):
        return query(self.goff, self.P, x, length, level, tau=float(self.hp[14]), grids=self.grids)

    def step_with_grad(self, grad, count=None):
        """The optimizer half of a step (C6) on a given normalised raw gradient [G][14]
        (e.g. the screen-space path's, next row f1); count: per-level sample counts (default:
        every level stepped).  Returns False for a no-op step."""
        g = _d(grad).reshape(-1, NP).copy()
        cnt = _i64(np.ones(self.L) if count is None else count)
        nonfinite = C.c_int64()
        r = lib().orc_opt_step(C.c_int(self.L), _p(self.goff, np.int64), _p(self.P, np.float64),
                               _p(self.M, np.float64), _p(self.V, np.float64),
                               _p(self.adam_step, np.int64), C.byref(self.t), _p(self.hp, np.float64),
                               _p(cnt, np.int64), _p(g, np.float64), C.byref(nonfinite))
        return r == 0


def chi2_3_cdf(x: float) -> float:
    """F_{chi^2_3}(x) = erf(sqrt(x/2)) - sqrt(2x/pi) e^{-x/2} (closed form, textbook)."""
    return math.erf(math.sqrt(x / 2.0)) - math.sqrt(2.0 * x / math.pi) * math.exp(-x / 2.0)


# ------------------------------------------------ screen-space evaluator (next row f1)
class _Cam(C.Structure):
    _fields_ = [("W", C.c_int), ("H", C.c_int), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("view", C.c_double * 12),
                ("znear", C.c_double)]


def _cam(cam):
    c = _Cam()
    c.W, c.H = int(cam["width"]), int(cam["height"])
    c.fx, c.fy, c.cx, c.cy = (float(cam[k]) for k in ("fx", "fy", "cx", "cy"))
    for i, v in enumerate(np.asarray(cam["view"], np.float64).reshape(12)):
        c.view[i] = float(v)
    c.znear = float(cam.get("znear", 0.2))
    return c


def project(P, cam):
    """orc_project of every row: [n][16] = ok, u, v, depth, conic(3), w, chat(3), x0, x1,
    y0, y1, rect_amb (screen_oracle.c, reading A23)."""
    P = _d(P).reshape(-1, NP)
    out = np.empty((len(P), 16))
    c = _cam(cam)
    for j in range(len(P)):
        lib().orc_project(_p(P[j].copy(), np.float64), C.byref(c), _p(out[j:j + 1], np.float64))
    return out


def render(P, cam, pix=None):
    """One level's cache image (sec.3.1, front-to-back alpha compositing of the
    projected Gaussians, reading A23): (rgb [H][W][3], T [H][W], amb [H][W]); with `pix`
    (linear pixel indices) only those pixels are computed (the rest is NaN)."""
    P = _d(P).reshape(-1, NP)
    c = _cam(cam)
    n = c.W * c.H
    rgb = np.full((n, 3), np.nan)
    T = np.full(n, np.nan)
    amb = np.zeros(n, np.int32)
    if pix is None:
        lib().orc_render(C.c_int64(len(P)), _p(P, np.float64), C.byref(c), C.c_int64(-1), None,
                         _p(rgb, np.float64), _p(T, np.float64), _p(amb, np.int32))
    else:
        pix = np.ascontiguousarray(pix, np.int64)
        lib().orc_render(C.c_int64(len(P)), _p(P, np.float64), C.byref(c), C.c_int64(len(pix)),
                         _p(pix, np.int64), _p(rgb, np.float64), _p(T, np.float64), _p(amb, np.int32))
    return rgb.reshape(c.H, c.W, 3), T.reshape(c.H, c.W), amb.reshape(c.H, c.W)


def image_loss(goff, P, cam, target, valid=None, denom=None, hdr_eps=0.01):
    """Eq. 4 over the per-level cache images: (total, per_level).  `denom` freezes
    the denominator images (reading A10's stop-gradient; its finite differences are the mode-0
    gradient)."""
    goff = _i64(goff)
    L = len(goff) - 1
    P = _d(P).reshape(-1, NP)
    c = _cam(cam)
    tgt = _d(target).reshape(-1)
    va = None if valid is None else np.ascontiguousarray(valid, np.uint8).reshape(-1)
    de = None if denom is None else _d(denom).reshape(-1)
    per = np.empty(L)
    lib().orc_image_loss.restype = C.c_double
    tot = lib().orc_image_loss(C.c_int(L), _p(goff, np.int64), _p(P, np.float64), C.byref(c),
                               _p(tgt, np.float64), None if va is None else _p(va, np.uint8),
                               None if de is None else _p(de, np.float64), C.c_double(hdr_eps),
                               _p(per, np.float64))
    return tot, per


def image_grad_fd(goff, P, cam, target, valid=None, hdr_eps=0.01, h=1e-6, mode=0):
    """Gradient of image_loss by fp64 central finite differences over every raw parameter:
    [G][14].  mode 0: denominators frozen at the unperturbed render (reading A10's stop-gradient);
    mode 1: the full quotient of Eq. 4 as written, denominators perturbed with the
    render.  Defines the screen-space backward for the tests (the derivative of the forward
    above, "inverse splatting")."""
    goff = _i64(goff)
    P = _d(P).reshape(-1, NP).copy()
    L = len(goff) - 1
    den = None if mode == 1 else np.concatenate([render(P[goff[l]:goff[l + 1]], cam)[0][None] for l in range(L)])
    g = np.zeros_like(P)
    for j in range(len(P)):
        for k in range(NP):
            v = P[j, k]
            step = h * max(1.0, abs(v))
            P[j, k] = v + step
            lp, _ = image_loss(goff, P, cam, target, valid, den, hdr_eps)
            P[j, k] = v - step
            lm, _ = image_loss(goff, P, cam, target, valid, den, hdr_eps)
            P[j, k] = v
            g[j, k] = (lp - lm) / (2 * step)
    return g

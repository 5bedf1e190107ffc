"""Round-2 parity cases (-m gpu), through the C ABI, against the fp64 oracle:

* the timed "lite" backward's coefficient gradients (gc_debug_coef_grads snapshot, the
  backward itself unchanged) and the raw gradients, at configs[2]'s full frame size, on the
  whole frame, against the culled oracle (SURVEY 8(c) gradient bar, both forms);
* the general path (rotated, anisotropic, scale LR > 0: north_star's "covariance factors") at
  full cfg2 size;
* finite samples far outside the culling grid (A17) mixed into border cells;
* culling-list overflow detected on the device under CUDA-graph replay, and list growth;
* Eq. 2 on degenerate levels (reading A20);
* the pageable-statistics ring with more than 64 calls in flight.
"""
import ctypes as C

import numpy as np
import pytest

import oracle
import workload
from test_gpu_parity import check_forward, check_grad_group, check_grads, cuda, grad_allow, make_cfg1, rows

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gsc():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2507_19718_b200 as m
    assert torch.cuda.is_available()
    return m


COEF_GROUPS = {"dmu": slice(0, 3), "dA": slice(3, 9), "dv": slice(9, 12)}


def check_coef(dev, st, ro, goff, what, lite_levels=(), allow=None):
    """Device coefficient gradients (unnormalised sums) vs the oracle's (normalised by
    1/(3 k_l)): every (level, coefficient group) under both gradient bars; on levels run by
    the lite backward (isotropic, scale group frozen) dA is exactly 0 on the device.
    ``allow``: oracle.grad_allowance()["coef"] (A3 boundary flips), or None."""
    for l in range(len(goff) - 1):
        sl = slice(goff[l], goff[l + 1])
        k = int(st.count[l])
        assert k == ro["count"][l]
        if k == 0:
            continue
        d = dev[sl].astype(np.float64) / (3.0 * k)
        for name, cs in COEF_GROUPS.items():
            if name == "dA" and l in lite_levels:
                assert np.all(dev[sl, cs] == 0.0), (what, l, "lite dA")
                continue
            check_grad_group(d[:, cs], ro["coef"][sl, cs], f"{what} level {l} {name}",
                             allow=None if allow is None else allow[sl, cs])


def allowance(c, P, x, ln, rgb, **kw):
    """Readings A3 + A21 per-element widening (test_gpu_parity.grad_allow)."""
    return grad_allow(c, P, x, ln, rgb, **kw)


def test_cfg2_full_frame_gradients_lite_and_raw(gsc):
    """configs[2], one full 1920x1080 frame (2,073,600 samples), default hyper-parameters:
    (1) the coefficient gradients of the timed lite backward, (2) the raw 14-parameter
    gradients (recording on), both against the culled oracle on the whole frame."""
    pos, alb = workload.init_cloud(2)
    counts = workload.CONFIGS[2]["counts"]
    x, ln, rgb = workload.fit_batch(2, frame=1)
    c = gsc.GSCache(counts, cuda(pos), cuda(alb), seed=2)
    c.reserve(len(x), 0)
    P = rows(c)
    ro = oracle.loss_grad(c.goff, P, x.astype(np.float64), ln, rgb.astype(np.float64), grids=c.grids())
    c.debug_enable_grads(False, coef=True)
    st = c.fit(cuda(x), cuda(ln), cuda(rgb))
    torch.cuda.synchronize()
    for l in range(4):
        assert abs(st.loss[l] - ro["loss"][l]) <= 1e-4 * ro["loss"][l]
    al = allowance(c, P, x, ln, rgb)
    dev = np.concatenate([c.debug_coef_grads(l) for l in range(4)])
    check_coef(dev, st, ro, c.goff, "cfg2 lite", lite_levels=(0, 1, 2, 3), allow=al["coef"])
    c2 = gsc.GSCache(counts, cuda(pos), cuda(alb), seed=2)
    c2.reserve(len(x), 0)
    c2.debug_enable_grads(True)
    st2 = c2.fit(cuda(x), cuda(ln), cuda(rgb))
    torch.cuda.synchronize()
    g = np.concatenate([c2.debug_grads_rows(l) for l in range(4)]).astype(np.float64)
    check_grads(g, ro["grad"], c2.goff, "cfg2 raw", iso_levels=(0, 1, 2, 3), allow=al["raw"])
    assert st2.n_pairs == st.n_pairs


def test_cfg2_full_frame_anisotropic_scale_lr(gsc):
    """The general (non-lite) path at full cfg2 size: every level rotated and anisotropic,
    scale LR 0.0125 (the paper's -CO variant): raw and coefficient gradients on the
    whole frame, then the first AdamW step of the scale group vs the oracle's."""
    pos, alb = workload.init_cloud(2)
    counts = workload.CONFIGS[2]["counts"]
    lr = [1.16e-3, 1e-3, 1.25e-2, 1.25e-2, 1.5e-1]
    hp = gsc.default_hparams(lr=lr)
    c = gsc.GSCache(counts, cuda(pos), cuda(alb), seed=2, hparams=hp)
    r = np.random.default_rng(31)
    for l in range(4):
        Pl = c.params_rows(l)
        Pl[:, 3:7] = r.normal(size=(len(Pl), 4)).astype(np.float32)
        Pl[:, 10:13] += r.uniform(-0.4, 0.2, (len(Pl), 3)).astype(np.float32)
        c.set_params_rows(l, Pl)
    x, ln, rgb = workload.fit_batch(2, frame=2)
    c.reserve(len(x), 0)
    P = rows(c)
    c.debug_enable_grads(True, coef=True)
    st = c.fit(cuda(x), cuda(ln), cuda(rgb))
    torch.cuda.synchronize()
    oc = oracle.OracleCache(counts, P, hp=dict(lr=lr), grids=c.grids())
    ro = oracle.loss_grad(c.goff, P, x.astype(np.float64), ln, rgb.astype(np.float64), grids=c.grids())
    oc.fit(x.astype(np.float64), ln, rgb.astype(np.float64))
    al = allowance(c, P, x, ln, rgb)
    g = np.concatenate([c.debug_grads_rows(l) for l in range(4)]).astype(np.float64)
    check_grads(g, ro["grad"], c.goff, "cfg2 aniso", allow=al["raw"])
    dev = np.concatenate([c.debug_coef_grads(l) for l in range(4)])
    check_coef(dev, st, ro, c.goff, "cfg2 aniso coef", allow=al["coef"])
    P1 = rows(c)
    # the scale group now steps: first AdamW step = -eta sign(g) wherever g is well above the
    # fp32 rounding level (test_first_step_matches_oracle_update's criterion)
    go = ro["grad"][:, 10:13]
    strong = np.abs(go) > 1e-3 * np.abs(go).max()
    d_dev, d_or = (P1 - P)[:, 10:13], (oc.P - P)[:, 10:13]
    assert strong.mean() > 0.5
    assert np.all(np.abs(d_dev - d_or)[strong] <= 1e-3 * 1.25e-2 + 4e-7 * (1 + np.abs(P[:, 10:13][strong])))


def test_far_outside_grid_samples(gsc):
    """Finite samples far outside a level's culling grid (x = +-5, +-1e3, +-1e30 on one or
    all axes) clamp into border cells (A17) and share work items with in-grid samples of those
    cells.  Lookups and gradients of every sample must match the oracle: the evaluators
    recentre on the cell's centre, not on an item's first sample."""
    c, _, _ = make_cfg1(gsc)
    P = rows(c)
    x, ln, rgb = workload.fit_batch(1, S=120_000, frame=5)
    r = np.random.default_rng(17)
    n_out = 6000
    far = r.choice([5.0, -5.0, 1e3, -1e3, 1e30, -1e30], size=(n_out, 3))
    keep = r.random((n_out, 3)) < 0.5                       # some axes stay in the grid
    far = np.where(keep, x[:n_out], far).astype(np.float32)
    far[keep.all(axis=1), 0] = 1e30
    idx = r.choice(len(x), n_out, replace=False)
    x[idx] = far
    # samples on the grid boundary region (border cells hold both kinds)
    y = c.query(cuda(x), cuda(ln)).cpu().numpy()
    yo, lv, _ = oracle.query(c.goff, P, x.astype(np.float64), ln, grids=c.grids())
    assert np.all(np.isfinite(y))
    check_forward(y, yo, P, c.goff, x, lv, what="outside-grid lookups")
    c.debug_enable_grads(True, coef=True)
    st = c.fit(cuda(x), cuda(ln), cuda(rgb))
    torch.cuda.synchronize()
    ro = oracle.loss_grad(c.goff, P, x.astype(np.float64), ln, rgb.astype(np.float64), grids=c.grids())
    for l in range(3):
        assert st.count[l] == ro["count"][l]
        assert abs(st.loss[l] - ro["loss"][l]) <= 1e-4 * ro["loss"][l]
    al = allowance(c, P, x, ln, rgb)
    g = np.concatenate([c.debug_grads_rows(l) for l in range(3)]).astype(np.float64)
    check_grads(g, ro["grad"], c.goff, "outside-grid", iso_levels=(0, 1, 2), allow=al["raw"])
    assert np.isfinite(rows(c)).all()


def test_overflow_detected_under_graph_replay(gsc):
    """Culling-list overflow is detected on the device: a CUDA-graph replay whose lists
    overflowed reports GC_FLAG_LISTS_OVERFLOWED and skips its optimizer step (no host code
    runs during replay).  The next eager call grows the lists (GC_ERR_STATE once, list
    generation + 1); the graph captured before the growth then runs on the grown lists (the
    kernels reach them through device state): no flag, a real step, lookups of the fitted
    cache equal to the oracle's."""
    c, _, _ = make_cfg1(gsc)
    x, ln, rgb = workload.fit_batch(1, S=50_000, frame=7)
    xd, lnd, rgbd = cuda(x), cuda(ln), cuda(rgb)
    c.reserve(len(x), 0)
    s = torch.cuda.Stream()
    st = gsc.pinned_stats()
    with torch.cuda.stream(s):
        c.fit(xd, lnd, rgbd, stream=s, stats=st)              # warm-up (eager)
    s.synchronize()
    assert st.flags == 0 and st.step == 1
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        c.fit(xd, lnd, rgbd, stream=s, stats=st)
    gen0 = c.list_generation()
    P0 = c.params_rows(0)
    P0[:, 10:13] = np.log(0.25)                                # ~10x the Eq. 2 extent
    c.set_params_rows(0, P0)                                   # its rebuild overflows
    before = rows(c)
    with torch.cuda.stream(s):
        g.replay()
    s.synchronize()
    assert st.flags == 1 and st.step == 0                      # detected without the host
    np.testing.assert_array_equal(rows(c), before)             # step skipped
    with pytest.raises(gsc.GCError) as ei:                     # eager: grow + rebuild, once
        c.fit(xd, lnd, rgbd)
    assert ei.value.status == 2
    assert c.list_generation() == gen0 + 1
    st2 = c.fit(xd, lnd, rgbd)
    torch.cuda.synchronize()
    assert st2.flags == 0 and st2.step >= 1
    with torch.cuda.stream(s):                                 # graph captured before the growth
        g.replay()
    s.synchronize()
    assert st.flags == 0 and st.step == st2.step + 1
    P = rows(c)
    xq, lq = workload.query_batch(1, S=20_000, frame=3)
    y = c.query(cuda(xq), cuda(lq)).cpu().numpy()
    yo, lv, _ = oracle.query(c.goff, P, xq.astype(np.float64), lq, grids=c.grids())
    check_forward(y, yo, P, c.goff, xq, lv, what="lookups after growth")


@pytest.mark.parametrize("kind", ["single", "coincident"])
def test_degenerate_level_eq2(gsc, kind):
    """Reading A20: a level of one point (counts[l] = 1) or of coincident points gets the
    absolute floor ln(0.5e-6) from Eq. 2 (NULL init scales), finite, equal to the oracle's;
    the cache then fits and answers lookups."""
    pos, alb = workload.init_cloud(1)
    pos, alb = pos[:256].copy(), alb[:256].copy()
    if kind == "coincident":
        pos[:] = pos[0]
    counts = [256, 1]
    c = gsc.GSCache(counts, cuda(pos), cuda(alb), seed=9)
    P = rows(c)
    Po = oracle.create(counts, pos.astype(np.float64), alb.astype(np.float64), seed=9)
    assert np.isfinite(P).all()
    np.testing.assert_allclose(P[:, 10:13], Po[:, 10:13].astype(np.float32), rtol=3e-7)
    x, ln, rgb = workload.fit_batch(1, S=5000)
    ln = np.minimum(ln, 2).astype(np.int32)
    y = c.query(cuda(x), cuda(ln)).cpu().numpy()
    yo, lv, _ = oracle.query(c.goff, P, x.astype(np.float64), ln, grids=c.grids())
    check_forward(y, yo, P, c.goff, x, lv, what=f"{kind} level")
    st = c.fit(cuda(x), cuda(ln), cuda(rgb))
    torch.cuda.synchronize()
    assert st.step == 1 and np.isfinite(rows(c)).all()


def test_pageable_stats_ring_many_in_flight(gsc):
    """More than the 64-slot ring of pageable statistics in flight without a synchronisation:
    every caller struct receives its own call's statistics."""
    c, _, _ = make_cfg1(gsc)
    x, ln, rgb = workload.fit_batch(1, S=4000, frame=9)
    xd, lnd, rgbd = cuda(x), cuda(ln), cuda(rgb)
    sts = []
    for k in range(150):
        stk = gsc.gc_fit_stats()                               # pageable
        n = 1000 + 17 * k
        c.fit(xd[:n], lnd[:n], rgbd[:n], stats=stk)
        sts.append((n, stk))
    torch.cuda.synchronize()
    for k, (n, stk) in enumerate(sts):
        assert stk.n_in == n and stk.step == k + 1, (k, stk.n_in, stk.step)


@pytest.mark.parametrize("mode", [1, 2])
def test_routed_modes_one_rank_through_nccl(gsc, mode):
    """gc_set_comm mode 1 (level-sharded) and mode 2 (owner-computes) on a one-rank
    communicator: every sample and lookup goes through the routing kernels (count, all-gather
    of the count matrix, pack, ncclSend/ncclRecv to itself, unpack; lookups back through the
    return exchange into caller order); mode 2 also through the owner / need-mask / boundary
    machinery (one slab: every Gaussian owned and interior) and the filtered list rebuild.
    Lookups (incl. invalid ones, a fixed level, host buffers), fit statistics, gradients and the
    first AdamW step are checked against the oracle on the caller's batch."""
    c, _, _ = make_cfg1(gsc)
    c.set_comm(gsc.nccl_unique_id(), 0, 1, mode=mode)
    info = c.comm_info()
    assert info["mode"] == mode and info["owned_levels"] == [0, 1, 2] and info["group_size"] == 1
    P = rows(c)
    xq, lq = workload.query_batch(1, S=30_001, frame=2)
    lq[::11] = 0
    xq[::13, 1] = np.nan
    y = c.query(cuda(xq), cuda(lq)).cpu().numpy()
    yo, lv, _ = oracle.query(c.goff, P, xq.astype(np.float64), lq, grids=c.grids())
    assert np.all(y[lv < 0] == 0) and (lv < 0).sum() > 0
    ok = lv >= 0
    check_forward(y[ok], yo[ok], P, c.goff, xq[ok], lv[ok], what=f"mode-{mode} lookups")
    y1 = c.query(xq[:5000], None, level=1)                          # host buffers, fixed level
    torch.cuda.synchronize()
    yo1, lv1, _ = oracle.query(c.goff, P, xq[:5000].astype(np.float64), np.full(5000, 2, np.int32),
                               grids=c.grids())
    ok1 = lv1 >= 0
    check_forward(np.asarray(y1)[ok1], yo1[ok1], P, c.goff, xq[:5000][ok1], lv1[ok1], what=f"mode-{mode} level 1")
    x, ln, rgb = workload.fit_batch(1, S=80_000, frame=3)
    x[::97, 2] = np.inf
    oc = oracle.OracleCache(c.counts, P, grids=c.grids())
    go = None
    c.debug_enable_grads(True)
    for step in range(2):
        Pb = rows(c)
        st = c.fit(cuda(x), cuda(ln), cuda(rgb))
        torch.cuda.synchronize()
        ro = oracle.loss_grad(c.goff, Pb, x.astype(np.float64), ln, rgb.astype(np.float64), grids=c.grids())
        assert st.n_in == len(x) and st.n_valid == int(ro["count"].sum()) and st.step == step + 1
        for l in range(3):
            assert st.count[l] == ro["count"][l]
            assert abs(st.loss[l] - ro["loss"][l]) <= 1e-4 * ro["loss"][l]
        g = np.concatenate([c.debug_grads_rows(l) for l in range(3)]).astype(np.float64)
        al = grad_allow(c, Pb, x, ln, rgb)
        check_grads(g, ro["grad"], c.goff, f"mode-{mode} step {step}", iso_levels=(0, 1, 2), allow=al["raw"])
        if step == 0:                  # the first AdamW step vs the oracle's (criterion of
            go = oc.fit(x.astype(np.float64), ln, rgb.astype(np.float64))["grad"]   # test_first_step...)
            P1 = rows(c)
            eta = np.array([1.16e-3] * 3 + [1e-3] * 4 + [1.25e-2] * 3 + [0.0] * 3 + [1.5e-1])
            strong = np.abs(go) > 1e-3 * np.abs(go).max(axis=0, keepdims=True)
            err = np.abs((P1 - P) - (oc.P - P))
            assert np.all(err[strong] <= 1e-3 * eta[np.nonzero(strong)[1]] + 4e-7 * (1 + np.abs(P[strong])))
            assert np.all(err <= 2.0 * eta[None, :] + 4e-7 * (1 + np.abs(P)))


def test_checkpoint_resume_equals_continuous(gsc):
    """gc_params + gc_adam_state after 3 fits, restored into a fresh cache (gc_set_params with
    reset_adam = 0, gc_set_adam_state incl. t, AdamW step counters and beta powers): the next
    3 fits reproduce the continuous run (up to float-atomic summation order), and
    the restored state reads back bit-exactly."""
    from test_gpu_parity import _close_up_to_atomic_order
    a, _, _ = make_cfg1(gsc)
    frames = [workload.fit_batch(1, S=60_000, frame=20 + f) for f in range(6)]
    for f in range(3):
        a.fit(*[cuda(v) for v in frames[f]])
    torch.cuda.synchronize()
    state = [(a.params_rows(l), *a.adam_state(l)) for l in range(3)]
    assert state[0][3]["t"] == 3 and state[0][3]["adam_step"][:3] == [3, 3, 3]
    b, _, _ = make_cfg1(gsc, seed=99)               # different init: everything must be restored
    for l, (p, m, v, ctr) in enumerate(state):
        b.set_params_rows(l, p)
        b.set_adam_state(l, m, v, ctr)
    for l, (p, m, v, ctr) in enumerate(state):
        p2, m2, v2, c2 = b.params_rows(l), *b.adam_state(l)
        np.testing.assert_array_equal(p2, p)
        np.testing.assert_array_equal(m2, m)
        np.testing.assert_array_equal(v2, v)
        assert c2 == ctr
    for f in range(3, 6):
        sa = a.fit(*[cuda(v) for v in frames[f]])
        sb = b.fit(*[cuda(v) for v in frames[f]])
        torch.cuda.synchronize()
        assert sa.step == sb.step == f + 1
        np.testing.assert_allclose(list(sb.loss[:3]), list(sa.loss[:3]), rtol=1e-5)
    _close_up_to_atomic_order(rows(b), rows(a))


def test_alg1_device_helper_bit_exact(gsc):
    """The device-callable Algorithm 1 helper (include/gscache_device.cuh, run by
    gc_alg1_terminate) vs oracle.alg1 on 20,000 random paths (1-8 vertices, C in [0.1, 4], q
    uniform, some q right at the 1 - Tr threshold): the termination decision, Tr_out and
    beta_{n+1} are fp32 operations in the same order on both sides, hence bit-exact."""
    r = np.random.default_rng(12)
    P, nmax = 20_000, 8
    sig = r.uniform(0.0, 1.0, (P, nmax, 3)).astype(np.float32)
    n = r.integers(0, nmax + 1, P).astype(np.int32)
    C_ = 1.7
    beta = r.uniform(0.05, 1.0, P).astype(np.float32)
    q = r.random(P).astype(np.float32)
    want = [oracle.alg1(sig[i], n[i], C_, beta[i], q[i], eps=1e-6) for i in range(P)]
    for i in range(0, P, 7):               # thresholds: q exactly 1 - Tr of the path
        _, _, bn = want[i]
        tr = np.float32(bn / beta[i]) if bn != beta[i] else None
        if tr is not None:
            q[i] = np.float32(1.0) - tr
            want[i] = oracle.alg1(sig[i], n[i], C_, beta[i], q[i], eps=1e-6)
    t, tro, bno = gsc.alg1_terminate(cuda(sig), cuda(n), C_, cuda(q), cuda(beta), eps=1e-6)
    torch.cuda.synchronize()
    t, tro, bno = t.cpu().numpy(), tro.cpu().numpy(), bno.cpu().numpy()
    np.testing.assert_array_equal(t, np.array([w[0] for w in want]))
    np.testing.assert_array_equal(tro, np.stack([w[1] for w in want]))
    np.testing.assert_array_equal(bno, np.array([w[2] for w in want], np.float32))
    assert 0.1 < t.mean() < 0.9


def test_reinit_equals_fresh_create(gsc):
    """gc_reinit (morphology change) on a cache that has been fitted: parameters,
    AdamW state, schedule, culling grids and lists afterwards are those of a fresh gc_create
    from the new cloud (bit-exact), and the caches then fit identically (up to atomic order)."""
    a, _, _ = make_cfg1(gsc)
    for f in range(2):
        a.fit(*[cuda(v) for v in workload.fit_batch(1, S=30_000, frame=40 + f)])
    torch.cuda.synchronize()
    r = np.random.default_rng(8)
    pos2 = (workload.init_cloud(1)[0][:4096] * 0.7 + r.normal(0, 0.02, (4096, 3))).astype(np.float32)
    alb2 = r.uniform(0.1, 0.9, (4096, 3)).astype(np.float32)
    a.reinit(cuda(pos2), alb2, seed=5)
    b = gsc.GSCache([4096, 1024, 256], pos2, alb2, seed=5)
    np.testing.assert_array_equal(rows(a), rows(b))
    for l in range(3):
        ma, va, ca = a.adam_state(l)
        assert not ma.any() and not va.any() and ca["t"] == 0 and ca["adam_step"][l] == 0
        for ga, gb in zip(a.grid(l), b.grid(l)):
            np.testing.assert_array_equal(ga, gb)
        oa, ia = a.debug_cull(l)
        ob, ib = b.debug_cull(l)
        np.testing.assert_array_equal(oa, ob)
        np.testing.assert_array_equal(ia, ib)
    Po = oracle.create([4096, 1024, 256], pos2.astype(np.float64), alb2.astype(np.float64), seed=5,
                       init_opacity=float(np.float32(0.1)), zcap=2.0, factor=0.5)
    np.testing.assert_array_equal(rows(a)[:, 0:10], Po.astype(np.float32).astype(np.float64)[:, 0:10])
    x = workload.fit_batch(1, S=30_000, frame=50)
    sa = a.fit(*[cuda(v) for v in x])
    sb = b.fit(*[cuda(v) for v in x])
    torch.cuda.synchronize()
    assert sa.step == sb.step == 1
    np.testing.assert_allclose(list(sa.loss[:3]), list(sb.loss[:3]), rtol=1e-6)

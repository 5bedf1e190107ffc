"""Row A8: dense all-pairs lookups on the tensor cores (gc_query_dense: tcgen05.mma kind::tf32,
3xTF32 split, recentred monomial features) against the fp64 oracle (-m gpu), under the
forward bar |dy| <= 1e-5 |y| + 1e-7 max|y| (north star: the tensor-core variant is allowed
"only if it stays inside the stated tolerance")."""
import numpy as np
import pytest

import oracle
import workload
from test_gpu_parity import check_forward, cuda, rows

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gsc():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2507_19718_b200 as m
    assert torch.cuda.is_available()
    return m


def dense_cache(gsc, tau, aniso=True, counts=(4096, 1024, 256)):
    pos, alb = workload.init_cloud(1)
    c = gsc.GSCache(list(counts), cuda(pos[:counts[0]]), cuda(alb[:counts[0]]), seed=7,
                    hparams=dict(cutoff_sigma=tau))
    if aniso:
        r = np.random.default_rng(11)
        P0 = c.params_rows(0)
        P0[:, 3:7] = r.normal(size=(len(P0), 4)).astype(np.float32)
        P0[:, 10:13] += r.uniform(-0.3, 0.3, (len(P0), 3)).astype(np.float32)
        c.set_params_rows(0, P0)
    return c


@pytest.mark.parametrize("tau,aniso", [(np.inf, True), (np.inf, False), (3.0, True)])
def test_dense_tc_lookups_match_oracle(gsc, tau, aniso):
    c = dense_cache(gsc, float(tau), aniso)
    P = rows(c)
    xq, lq = workload.query_batch(1, S=12_001, frame=6)
    lq[::19] = 0                                                  # invalid -> 0
    y = c.query_dense(cuda(xq), cuda(lq)).cpu().numpy()
    yo, lv, _ = oracle.query(c.goff, P, xq.astype(np.float64), lq, tau=float(tau),
                             grids=None if not np.isfinite(tau) else c.grids())
    assert np.all(y[lv < 0] == 0)
    ok = lv >= 0
    check_forward(y[ok], yo[ok], P, c.goff, xq[ok], lv[ok], tau=float(tau), what=f"dense tc tau={tau}")


def test_dense_tc_fixed_level_and_ragged(gsc):
    c = dense_cache(gsc, float("inf"))
    P = rows(c)
    for S in (1, 127, 129, 3000):
        xq, _ = workload.query_batch(1, S=S, frame=S)
        y = c.query_dense(cuda(xq), None, level=2).cpu().numpy()
        yo, lv, _ = oracle.query(c.goff, P, xq.astype(np.float64), None, level=2, tau=float("inf"))
        check_forward(y, yo, P, c.goff, xq, lv, tau=float("inf"), what=f"dense tc S={S}")


def _dense_fit_case(gsc, n0, S, seed):
    r = np.random.default_rng(seed)
    pos = r.uniform(-0.8, 0.8, (n0, 3)).astype(np.float32)
    alb = r.uniform(0.2, 0.9, (n0, 3)).astype(np.float32)
    ls = np.full((n0, 3), np.log(0.3), np.float32)
    hp = gsc.default_hparams(cutoff_sigma=float("inf"))
    c = gsc.GSCache([n0, max(n0 // 4, 1)], pos, alb, init_log_scale=ls, seed=1, hparams=hp)
    P0 = c.params_rows(0)
    P0[:, 3:7] = r.normal(size=(n0, 4)).astype(np.float32)
    P0[:, 10:13] += r.uniform(-0.3, 0.3, (n0, 3)).astype(np.float32)
    c.set_params_rows(0, P0)
    x = r.uniform(-0.9, 0.9, (S, 3)).astype(np.float32)
    ln = r.integers(1, 3, S).astype(np.int32)
    rgb = r.uniform(0, 2, (S, 3)).astype(np.float32)
    return c, x, ln, rgb


@pytest.mark.parametrize("n0,S", [(64, 3000), (448, 3000), (1000, 9000)])
def test_dense_fit_gradients_match_oracle(gsc, n0, S):
    """gc_fit_dense (row A8's backward: Q^T and E^T . [g phi, g] as two chained tcgen05
    products, the second with its A operand in tensor memory) against the fp64 oracle's
    loss_grad at tau = infinity: per-level loss and valid counts, and all 14 raw gradients
    under both gradient bars (with reading A21's summation-order allowance); sizes span one
    and several 128-Gaussian chunks, ragged work items and both levels."""
    from test_gpu_parity import check_grads, grad_allow
    c, x, ln, rgb = _dense_fit_case(gsc, n0, S, seed=n0)
    x[::97] = np.nan                                          # dropped samples
    rgb[5::89] = np.inf
    P = rows(c)
    c.debug_enable_grads(True)
    c.profile_enable(True)
    st = c.fit_dense(cuda(x), cuda(ln), cuda(rgb))
    torch.cuda.synchronize()
    prof = c.profile_read()
    c.profile_enable(False)
    assert {"dense_tc", "dense_loss", "dense_bwd", "adamw"} <= set(prof) and "fwdbwd" not in prof, prof
    keep = np.isfinite(x).all(1) & np.isfinite(rgb).all(1)
    xo, lo_, ro_ = x[keep], ln[keep], rgb[keep]
    ro = oracle.loss_grad(c.goff, P, xo.astype(np.float64), lo_, ro_.astype(np.float64), tau=np.inf)
    for l in range(2):
        assert st.count[l] == ro["count"][l]
        assert abs(st.loss[l] - ro["loss"][l]) <= 1e-4 * ro["loss"][l]
    g = np.concatenate([c.debug_grads_rows(l) for l in range(2)]).astype(np.float64)
    al = grad_allow(c, P, xo, lo_, ro_, tau=np.inf, brute=True)
    check_grads(g, ro["grad"], c.goff, f"dense fit n0={n0}", iso_levels=(1,), allow=al["raw"])


def test_dense_fit_steps_track_world_fit(gsc):
    """Five gc_fit_dense steps and five gc_fit steps (tau = infinity, same frames) from the same
    cache: per-level losses agree at every step (the same method, two evaluators) and the
    parameters stay within Adam's amplification of last-bit gradient differences."""
    from test_gpu_parity import _close_up_to_atomic_order
    c1, x, ln, rgb = _dense_fit_case(gsc, 300, 4000, seed=3)
    c2, _, _, _ = _dense_fit_case(gsc, 300, 4000, seed=3)
    for k in range(5):
        s1 = c1.fit_dense(cuda(x), cuda(ln), cuda(rgb))
        torch.cuda.synchronize()
        l1 = list(s1.loss[:2])
        s2 = c2.fit(cuda(x), cuda(ln), cuda(rgb))
        torch.cuda.synchronize()
        np.testing.assert_allclose(l1, list(s2.loss[:2]), rtol=1e-4)
    _close_up_to_atomic_order(rows(c1), rows(c2))


def test_dense_fit_fixed_level_and_cutoff(gsc):
    """gc_fit_dense with a fixed level (path_len NULL: every sample on level 0) and with the
    cut-off tau = 3 (the backward masks e by Q <= tau^2 like the forward): gradients against the
    oracle's loss_grad under both bars, with reading A3's boundary allowance for tau = 3."""
    from test_gpu_parity import check_grads, grad_allow
    c, x, ln, rgb = _dense_fit_case(gsc, 448, 3000, seed=77)
    P = rows(c)
    c.debug_enable_grads(True)
    c.fit_dense(cuda(x), None, cuda(rgb), level=0)
    torch.cuda.synchronize()
    ln0 = np.ones(len(x), np.int32)
    g = np.concatenate([c.debug_grads_rows(l) for l in range(2)]).astype(np.float64)
    ro = oracle.loss_grad(c.goff, P, x.astype(np.float64), ln0, rgb.astype(np.float64), tau=np.inf)
    assert np.abs(g[c.goff[1]:]).max() == 0.0                 # level 1 untouched
    al = grad_allow(c, P, x, ln0, rgb, tau=np.inf, brute=True)
    n0 = c.goff[1]
    check_grads(g[:n0], ro["grad"][:n0], [0, n0], "dense fit fixed level", allow=al["raw"][:n0])
    # tau = 3
    r = np.random.default_rng(5)
    pos = r.uniform(-0.8, 0.8, (448, 3)).astype(np.float32)
    alb = r.uniform(0.2, 0.9, (448, 3)).astype(np.float32)
    ls = np.full((448, 3), np.log(0.3), np.float32)
    c3 = gsc.GSCache([448, 112], pos, alb, init_log_scale=ls, seed=1, hparams=dict(cutoff_sigma=3.0))
    P3 = rows(c3)
    c3.debug_enable_grads(True)
    c3.fit_dense(cuda(x), cuda(ln), cuda(rgb))
    torch.cuda.synchronize()
    g3 = np.concatenate([c3.debug_grads_rows(l) for l in range(2)]).astype(np.float64)
    ro3 = oracle.loss_grad(c3.goff, P3, x.astype(np.float64), ln, rgb.astype(np.float64), tau=3.0, grids=c3.grids())
    # every sample meets ~100 Gaussians inside 3 sigma, so ~2 % of the samples hold a pair within
    # 1e-4 tau^2 of the cut-off (reading A3); those get the allowance
    al3 = grad_allow(c3, P3, x, ln, rgb, tau=3.0, max_amb_rate=0.05)
    check_grads(g3, ro3["grad"], c3.goff, "dense fit tau=3", iso_levels=(0, 1), allow=al3["raw"])


def test_dense_fit_empty_and_all_invalid(gsc):
    """gc_fit_dense with no samples and with only dropped samples (non-finite positions, n < 1,
    non-finite colours): k_l = 0 on every level, so no optimizer step -- parameters unchanged."""
    c, x, ln, rgb = _dense_fit_case(gsc, 200, 300, seed=9)
    P = rows(c)
    st = c.fit_dense(cuda(x[:0]), cuda(ln[:0]), cuda(rgb[:0]))
    torch.cuda.synchronize()
    assert st.count[0] == 0 and st.count[1] == 0
    x[:100] = np.nan
    ln[100:200] = 0
    rgb[200:] = np.nan
    st = c.fit_dense(cuda(x), cuda(ln), cuda(rgb))
    torch.cuda.synchronize()
    assert st.count[0] == 0 and st.count[1] == 0 and st.loss[0] == 0.0
    np.testing.assert_array_equal(rows(c), P)

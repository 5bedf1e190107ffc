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

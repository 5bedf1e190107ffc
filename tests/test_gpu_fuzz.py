"""A short randomised soak of the public API (tests/fuzz_api.py): random sequences of fit,
query, fit_query (deferred step on and off), dense lookups and fits, screen render / fit,
parameter and Adam-state round trips, reinit and new caches, inputs of random sizes including
0 with dropped samples; no call may fail, and every tenth call a query is compared with the
fp64 oracle on the library's current parameters (loose 1e-3 bar: this checks state, not
numerics -- the parity tests do that)."""
import pytest

pytestmark = pytest.mark.gpu


def test_api_soak():
    torch = pytest.importorskip("torch")
    import __graft_entry__
    __graft_entry__.build()
    assert torch.cuda.is_available()
    import fuzz_api
    res = fuzz_api.run(calls=200, seed=11)
    assert res["worst_query_rel_err"] < 1e-3
    assert len(res["per_op"]) >= 10

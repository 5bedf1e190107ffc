"""The C-ABI library loads and exports every symbol include/gscache.h declares (no compute
calls: these run on the CPU box without a GPU)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def built():
    from paper_2507_19718_b200 import build
    return build.build()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "gscache.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gc_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_binding_exports():
    import paper_2507_19718_b200 as pkg
    assert header_symbols() == sorted(pkg.EXPORTS)


def test_library_exports_every_declared_symbol(built):
    out = subprocess.run(["nm", "-D", "--defined-only", built], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (gc_[a-z_0-9]+)$", out, flags=re.M))
    missing = set(header_symbols()) - exported
    assert not missing, missing


def test_library_loads_and_binds(built):
    import paper_2507_19718_b200 as pkg
    L = pkg.lib()
    for name in pkg.EXPORTS:
        assert hasattr(L, name)
    hp = pkg.default_hparams()
    assert abs(hp.lr[0] - 1.16e-3) < 1e-9 and hp.lr[3] == 0.0 and abs(hp.cutoff_sigma - 3) < 1e-7
    assert L.gc_status_string(1) == b"GC_ERR_ARG"


def test_arg_errors_have_no_side_effects(built):
    """Host-checked argument errors return GC_ERR_ARG before touching any device."""
    import ctypes as C

    import numpy as np

    import paper_2507_19718_b200 as pkg
    L = pkg.lib()
    h = C.c_void_p()
    counts = np.array([10, 20], np.int64)                      # increasing -> error
    pos = np.zeros((10, 3), np.float32)
    assert L.gc_create(2, counts.ctypes.data, pos.ctypes.data, pos.ctypes.data, None, 0, None, 0,
                       C.byref(h)) == 1
    assert b"non-increasing" in L.gc_last_error()
    assert L.gc_create(0, counts.ctypes.data, pos.ctypes.data, pos.ctypes.data, None, 0, None, 0,
                       C.byref(h)) == 1
    assert L.gc_fit(None, None, None, None, 0, None, None) == 1
    # the round-2 entry points: a NULL handle is GC_ERR_ARG before any device work
    assert L.gc_fit_dense(None, None, None, 0, None, 0, None, None) == 1
    assert L.gc_query_dense(None, None, None, 0, 0, None, None) == 1
    assert L.gc_render(None, None, -1, None, None, None) == 1
    assert L.gc_fit_image(None, None, None, None, None, None) == 1


def test_sources_are_sm100a_only():
    from paper_2507_19718_b200 import build
    import inspect
    src = inspect.getsource(build)
    assert "arch=compute_100a,code=sm_100a" in src


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2507_19718_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "gscache_oracle" not in txt, f

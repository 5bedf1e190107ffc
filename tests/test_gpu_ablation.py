"""The stability ablation of next row f4 (App. A.2: -REG, -CO, -SC), short
protocol, through the library on the GPU (-m gpu), in both the world-space fit (gc_fit) and
the paper's own screen-space fit (gc_fit_image, row f1): every variant stays finite and
learns (held-out error falls from its first evaluation), the frozen scale group of the paper
default is untouched (reading A16) while -CO moves it.  tools/ablation.py runs the full
protocol (profiles/*ablation*.json, DESIGN 6.2)."""
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


@pytest.fixture(scope="module")
def abl():
    import __graft_entry__
    __graft_entry__.build()
    import ablation
    return ablation


@pytest.mark.parametrize("path", ["world", "screen"])
def test_ablation_variants_stable_and_learning(abl, path):
    dev = torch.device("cuda", 0)
    frames = 24
    res = {}
    for name, over in abl.VARIANTS.items():
        r = (abl.run_screen(1, frames, name, over, dev) if path == "screen"
             else abl.run(1, frames, name, over, dev, 0.0))
        res[name] = r
        assert not r["nonfinite"], (path, name)
        first, last = r["curve"][0][1], r["curve"][-1][1]
        assert last < first, (path, name, first, last)
    import workload
    pos, _ = workload.init_cloud(1)
    assert res["-CO"]["max_extent_es"] != res["ours"]["max_extent_es"]

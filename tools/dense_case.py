"""The A8 dense case of bench.py (cfg1 levels, tau = inf, anisotropic level 0, 262,144 lookups)
run a few times for ncu: python tools/dense_case.py [tc|cuda]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2507_19718_b200 as gsc  # noqa: E402


class A:
    steps = 6


if __name__ == "__main__":
    dev = torch.device("cuda", 0)
    print(bench.dense_bench(gsc, dev, 0, A()))

"""bench.py's screen-space leg alone (cfg2 cache, 1920x1080): python tools/screen_case.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2507_19718_b200 as gsc  # noqa: E402


class A:
    steps = int(os.environ.get("STEPS", "24"))


if __name__ == "__main__":
    r = bench.screen_bench(gsc, 2, torch.device("cuda", 0), 0, A())
    print(round(r["render_ms"] * 1e3, 1), round(r["fit_image_ms"] * 1e3, 1))

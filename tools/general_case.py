"""bench.py's general-path leg alone (cfg2 frames, every level rotated + anisotropic, scale LR
0.0125): frame time, and the per-kernel device times of eager serialised frames.
  python tools/general_case.py [--aniso-only]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2507_19718_b200 as gsc  # noqa: E402
import workload  # noqa: E402


class A:
    steps = 20
    warmup = 5
    no_defer = False
    no_graph = False
    cell_scale = 1.0


if __name__ == "__main__":
    dev = torch.device("cuda", 0)
    frames, S = bench.make_frames(2, 0, 1, 4, False, False, dev)
    outq = torch.empty((S, 3), dtype=torch.float32, device=dev)
    stream = torch.cuda.Stream(device=dev)

    def frame_call(cch, x, ln, rgb, xq, lq, out, s_):
        return cch.fit_query(x, ln, rgb, xq, lq, out=out, stream=s_)[1]
    r = bench.general_bench(gsc, 2, dev, 0, A(), frames, S, outq, stream, frame_call)
    print(r)

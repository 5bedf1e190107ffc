"""N-rank NCCL paths of the library on real GPUs (-m gpu; skipped below 2 GPUs).

Each case launches tests/mr_worker.py under torchrun with 2 ranks: data parallel (mode 0),
level-sharded (mode 1), spatial owner-computes (mode 2) and ZeRO data parallel (mode 3), each
checked on rank 0 against the one-rank oracle on the concatenated batch (C9).  The single-GPU boxes of this run skip them; the one-rank NCCL
paths (mode 0 identity, mode 1 routed through itself) run in test_gpu_parity*.py."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("mode", [0, 1, 2, 3])
def test_two_rank_matches_one_rank_oracle(mode):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    import __graft_entry__
    __graft_entry__.build()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + mode),
           os.path.join(ROOT, "tests", "mr_worker.py"), str(mode)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]

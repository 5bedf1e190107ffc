"""Host<->device copy bandwidth of this box (pinned buffers, 91 MB = one cfg2 frame's inputs):
context for bench.py's e2e number.  python tools/pcie_peak.py"""
import torch

n = 91_238_400 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
h2 = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
d2 = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()


def timed(fn, reps=20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


h2d = timed(lambda: d.copy_(h, non_blocking=True))
d2h = timed(lambda: h2.copy_(d, non_blocking=True))


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


dup = timed(both)
gb = n * 4 / 1e9
print({"bytes": n * 4, "h2d_GBps": gb / (h2d * 1e-3), "d2h_GBps": gb / (d2h * 1e-3),
       "duplex_h2d_GBps": gb / (dup * 1e-3)})

"""Per-kernel summary of the screen-space leg's ncu launch list (tools/screen_ncu.sh or
tools/screen_ab.sh -> gpurun_out/screen_launches.csv): median device time and DRAM bytes per
launch of every kernel of gc_render / gc_fit_image, and the per-call sums.
  python tools/screen_summary.py gpurun_out/screen_launches.csv > profiles/r02_screen_launches.md"""
import collections
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import launches  # noqa: E402

L = list(launches(sys.argv[1]).items())
# calls: a render is k_sproject .. k_sraster; a fit adds k_stats .. k_cull_emit
calls, cur = [], None
for (i, n), m in L:
    name = n.split("::")[-1]
    if name == "k_sproject":
        cur = []
        calls.append(cur)
    if cur is not None:
        cur.append((name, m.get("gpu__time_duration.sum", 0.0),
                    (m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)) / 1e6))
fits = [c for c in calls if any(k == "k_sraster_bwd" for k, _, _ in c)]
renders = [c for c in calls if c not in fits]


def table(cs, title):
    per = collections.OrderedDict()
    for c in cs[1:] or cs:            # skip the first call (buffer growth)
        for k, us, mb in c:
            per.setdefault(k, []).append((us, mb))
    ncall = max(len(cs) - 1, 1)
    print(f"\n### {title} ({ncall} calls, median per launch)\n")
    print("| kernel | launches/call | us | DRAM MB |")
    print("|---|---|---|---|")
    tot = 0.0
    for k, v in per.items():
        us = statistics.median(x for x, _ in v)
        mb = statistics.median(y for _, y in v)
        lpc = len(v) / ncall
        tot += us * lpc
        print(f"| {k} | {lpc:.0f} | {us:.1f} | {mb:.2f} |")
    print(f"| **sum** | | **{tot:.1f}** | |")


print("# Screen-space leg (f1) launch list, cfg2 cache at 1920x1080, 4 levels")
print("\nncu `--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
      "--clock-control none` over `tools/screen_case.py` (cold-cache, serialised launches).")
table(renders, "gc_render")
table(fits, "gc_fit_image")

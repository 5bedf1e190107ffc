"""Markdown summary of every kernel in an `ncu --set full` report (key metrics + stall reasons):
  python tools/ncu_kernel_md.py REPORT.ncu-rep "title" ["note"]"""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__inst_executed.avg.per_cycle_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum"]
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
print(f"# {sys.argv[2]}\n")
if len(sys.argv) > 3:
    print(sys.argv[3] + "\n")
print(f"Source: `{sys.argv[1].split('/')[-1]}` (ncu --set full --clock-control none).\n")
for r in rows[2:]:
    d = dict(zip(h, r))
    print(f"## {d['Kernel Name'].split('(')[0]}\n")
    print("| metric | value |\n|---|---|")
    for k in KEYS:
        if k in d:
            print(f"| {k} | {d[k]} |")
    st = [(k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), d[k])
          for k in h if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")]
    st = [(k, float(v)) for k, v in st if v not in ("", "n/a")]
    print("\n| stall (warps per issue) | value |\n|---|---|")
    for k, v in sorted(st, key=lambda x: -x[1]):
        if v > 0.1:
            print(f"| {k} | {v:.2f} |")
    print()

"""Summarise an ncu launch list (csv) + a --set full report into profiles/ markdown/json."""
import collections
import csv
import json
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == 'ID'][0]
    h = rows[hi]
    out = collections.OrderedDict()
    for r in rows[hi + 1:]:
        d = dict(zip(h, r))
        key = (int(d['ID']), d['Kernel Name'].split('(')[0])
        unit = d.get('Metric Unit', '')
        v = float(d['Metric Value'].replace(',', ''))
        if unit == 'nsecond' or unit == 'ns':
            v /= 1e3
        elif unit == 'msecond':
            v *= 1e3
        if unit in ('Kbyte', 'KB'):
            v *= 1e3
        elif unit in ('Mbyte', 'MB'):
            v *= 1e6
        elif unit in ('Gbyte', 'GB'):
            v *= 1e9
        out.setdefault(key, {})[d['Metric Name']] = v
    return out


def main(csv_path, rep_path, tag):
    L = launches(csv_path)
    per = collections.defaultdict(lambda: [0, 0.0, 0.0])
    # everything launched before the first step's k_keys belongs to gc_create; torch fills too
    first = min((i for (i, name) in L if "k_keys" in name), default=0)
    # the bench's later legs (screen space f1, general path, dense A8) launch some of the same
    # kernels (k_stats, k_adamw, the culling rebuild): stop at the first launch of those legs
    last = min((i for (i, name) in L if any(k in name for k in ("k_sproject", "k_dense_tc", "k_sraster"))),
               default=1 << 60)
    frame = ("k_keys", "k_scan", "k_scatter", "k_fwdbwd", "k_query", "k_stats", "k_step_scalars", "k_adamw",
             "k_record_cull", "k_cull_emit")
    for (i, name), m in L.items():
        if i < first or i >= last or name.startswith("at::") or "at::" in name:
            continue
        if not any(name.endswith(f) for f in frame):     # the bench's screen (f1) / dense (A8) legs
            continue
        p = per[name]
        p[0] += 1
        p[1] += m.get('gpu__time_duration.sum', 0.0)
        p[2] += m.get('dram__bytes_read.sum', 0.0) + m.get('dram__bytes_write.sum', 0.0)
    tot = sum(v[1] for v in per.values())
    lines = [f"# ncu launch list summary ({tag})", "",
             "Cold-cache, serialised per-launch times from `ncu --metrics gpu__time_duration.sum,"
             "dram__bytes_read.sum,dram__bytes_write.sum --clock-control none` over the bench command "
             "(compare SHARES, not absolutes).  Launches before the first step (gc_create: Eq. 2 kNN, first "
             "culling build), torch fills and the bench's separate screen-space (f1) and dense (A8) legs are "
             "excluded: shares are of the fit+query frame kernels.", "",
             "| kernel | launches | mean us | share | DRAM MB/launch |", "|---|---|---|---|---|"]
    traffic = {}
    for name, (n, t, b) in sorted(per.items(), key=lambda x: -x[1][1]):
        lines.append(f"| {name} | {n} | {t / n:.1f} | {t / tot * 100:.1f}% | {b / n / 1e6:.2f} |")
        traffic[name] = b / n
    if rep_path:
        raw = subprocess.run(["ncu", "-i", rep_path, "--page", "raw", "--csv", "--metrics",
                              "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
                              "sm__throughput.avg.pct_of_peak_sustained_elapsed,"
                              "sm__warps_active.avg.pct_of_peak_sustained_active,"
                              "smsp__inst_executed.sum,sm__inst_executed.avg.per_cycle_active,"
                              "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,"
                              "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,"
                              "launch__registers_per_thread,lts__t_sectors_op_red.sum"],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(raw.splitlines()))
        h = rows[0]
        lines += ["", f"## `ncu --set full` ({rep_path.split('/')[-1]})", "",
                  "| kernel | " + " | ".join(c.split('__')[1] for c in h if '__' in c) + " |",
                  "|---|" + "---|" * len([c for c in h if '__' in c])]
        issue = {}
        for r in rows[2:]:
            d = dict(zip(h, r))
            lines.append(f"| {d['Kernel Name'].split('(')[0]} | " + " | ".join(d[c] for c in h if '__' in c) + " |")
            name = d['Kernel Name'].split('(')[0].replace('void ', '').split('<')[0]
            try:
                issue.setdefault(name, {"ipc": float(d['sm__inst_executed.avg.per_cycle_active']),
                                        "fma_pipe_pct": float(d['sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active']),
                                        "xu_pipe_pct": float(d['sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active'])})
            except (KeyError, ValueError):
                pass
        json.dump({"source": f"{tag} ncu --set full ({rep_path.split('/')[-1]}): sm__inst_executed.avg.per_cycle_active "
                             "(issue peak 4 per SM per cycle), FMA / XU pipe utilisation",
                   "kernels": issue}, open("profiles/issue.json", "w"), indent=1)
    print("\n".join(lines))
    json.dump({"source": f"{tag} ncu launch list (dram__bytes_read.sum + dram__bytes_write.sum, mean per launch)",
               "bytes_per_launch": traffic}, open("profiles/traffic.json", "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None, sys.argv[3] if len(sys.argv) > 3 else "r01")

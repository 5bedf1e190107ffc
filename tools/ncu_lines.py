"""Aggregate an ncu source page (cuda,sass csv) per CUDA source line: inst share, stall share."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[2]
iE = h.index('Instructions Executed'); iS = h.index('Warp Stall Sampling (All Samples)')
stall_cols = [i for i, n in enumerate(h) if n.startswith('stall_') and 'Not Issued' not in n]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


cur = None; agg = {}; src = {}; fname = None; reasons = {}
for r in rows:
    if len(r) < 2:
        continue
    if r[0] == 'File Path':
        fname = r[1]; continue
    if r[0].isdigit():
        cur = (fname, int(r[0])); src[cur] = r[1]
    elif cur and r[2:3] and r[2].startswith('0x'):
        a = agg.setdefault(cur, [0, 0, {}]); a[0] += f(r[iE]); a[1] += f(r[iS])
        for i in stall_cols:
            a[2][h[i]] = a[2].get(h[i], 0) + f(r[i]); reasons[h[i]] = reasons.get(h[i], 0) + f(r[i])
tot = sum(v[0] for v in agg.values()); totS = sum(v[1] for v in agg.values())
print('warp-inst', tot, 'stall samples', totS)
for k, v in sorted(reasons.items(), key=lambda x: -x[1])[:8]:
    print(f"  {k} {v / totS * 100:.1f}%")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
key = 1 if (len(sys.argv) > 3 and sys.argv[3] == 'stall') else 0
for k, v in sorted(agg.items(), key=lambda x: -x[1][key])[:n]:
    top = sorted(v[2].items(), key=lambda x: -x[1])[:2]
    print(f"{(k[0] or '?').split('/')[-1][:10]}:{k[1]:>4} {v[0] / tot * 100:5.1f}% inst {v[1] / max(totS, 1) * 100:5.1f}% stall "
          f"{[(a[6:], round(b / max(totS, 1) * 100, 1)) for a, b in top]} {src[k].strip()[:70]}")

"""Top stall lines of one kernel's SASS source page: python tools/ncu_src.py rep.ncu-rep regex [frac]"""
import csv
import io
import subprocess
import sys

rep, rx = sys.argv[1], sys.argv[2]
frac = float(sys.argv[3]) if len(sys.argv) > 3 else 0.012
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                      f"regex:{rx}", "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
ends = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
block = rows[ends[0] + 1:(ends[1] if len(ends) > 1 else len(rows))]
hdr, data = block[0], block[1:]
ia, ss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[ss] or 0) for r in data)
print("samples", tot, "instructions", sum(int(r[ia] or 0) for r in data), "sass lines", len(data))
for i, r in enumerate(data):
    if int(r[ss] or 0) > tot * frac:
        print(f"{i:5d} {r[ss]:>6s} {r[ia]:>9s}  {r[1].strip()[:90]}")

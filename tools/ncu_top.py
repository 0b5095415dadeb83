"""Top warp-stall instructions of an ncu --set full report (SASS source page).
  python tools/ncu_top.py report.ncu-rep [n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
nshow = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(out)))
hi = [i for i, x in enumerate(r[:3]) if "Address" in x][0]
h, rows = r[hi], r[hi + 1:]
ix = {k: i for i, k in enumerate(h)}
S = "Warp Stall Sampling (All Samples)"


def f(x, k):
    try:
        return float(x[ix[k]] or 0)
    except (ValueError, KeyError):
        return 0.0


tot = sum(f(x, S) for x in rows)
order = {id(x): n for n, x in enumerate(rows)}
for x in sorted(rows, key=lambda x: -f(x, S))[:nshow]:
    print(f"{f(x, S) / tot * 100:5.1f}% #{order[id(x)]:5d} {x[ix['Source']][:70]:70s} exe {x[ix['Instructions Executed']]}")

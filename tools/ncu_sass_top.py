"""Top SASS instructions of a one-kernel ncu report by stall samples and by
executed instructions: python tools/ncu_sass_top.py rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(out)))
hi = [i for i, x in enumerate(r[:3]) if "Address" in x][0]
h, rows = r[hi], r[hi + 1:]
ia, isrc, ismp = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
recs = []
for x in rows:
    try:
        recs.append((float(x[ismp] or 0), float(x[ia] or 0), x[h.index("Address")], x[isrc]))
    except (ValueError, IndexError):
        pass
ts = sum(a[0] for a in recs) or 1
ti = sum(a[1] for a in recs) or 1
print(f"total samples {ts:.0f}, warp instructions {ti:.4g}")
for s, n, a, src in sorted(recs, key=lambda t: -t[0])[:top]:
    print(f"{s / ts * 100:7.3f}% smp {n / ti * 100:7.3f}% inst {a} {src}")

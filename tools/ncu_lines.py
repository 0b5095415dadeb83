"""Per-CUDA-source-line instruction / stall-sample breakdown of an ncu report
(--import-source on, -lineinfo).  Usage: python tools/ncu_lines.py rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = "?"
hdr = None
recs = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0] or len(r) < len(hdr) - 5:
        continue
    ie = hdr.index("Instructions Executed")
    sm = hdr.index("Warp Stall Sampling (All Samples)")
    try:
        n = float(r[ie]); s = float(r[sm])
    except ValueError:
        continue
    recs.append((n, s, fname, int(r[0]), r[1].strip()))
tot = sum(x[0] for x in recs) or 1
tots = sum(x[1] for x in recs) or 1
recs.sort(key=lambda x: -x[0])
print(f"total inst {tot:.4g}  samples {tots:.4g}")
for n, s, f, ln, src in recs[:top]:
    print(f"{n / tot * 100:5.1f}% inst {s / tots * 100:5.1f}% smp  {f}:{ln:<5d} {src[:90]}")

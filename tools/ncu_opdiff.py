"""Per-opcode warp instructions per 32 particles of two ncu reports (SASS
source page), largest differences first: python tools/ncu_opdiff.py A B n."""
import collections
import csv
import io
import subprocess
import sys


def ops(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hi = [i for i, x in enumerate(r[:3]) if "Address" in x][0]
    h, rows = r[hi], r[hi + 1:]
    ia, isrc = h.index("Instructions Executed"), h.index("Source")
    c = collections.Counter()
    for x in rows:
        n = float(x[ia] or 0)
        t = x[isrc].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        c[op] += n
    return c


a, b = ops(sys.argv[1]), ops(sys.argv[2])
scale = 32.0 / float(sys.argv[3])
keys = sorted(set(a) | set(b), key=lambda k: -abs(a[k] - b[k]))
for k in keys[:25]:
    print(f"{k:28s} {a[k] * scale:8.2f} {b[k] * scale:8.2f} {(a[k] - b[k]) * scale:+8.2f}")

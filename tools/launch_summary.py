"""Aggregates an ncu gpu__time_duration launch list per kernel (share of the
total device time; ncu launches are cold-cache and serialised, so compare
shares, not absolutes)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if len(r) > 5 and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[hdr.index("Metric Name")] == "gpu__time_duration.sum":
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
        ns = float(r[hdr.index("Metric Value")].replace(",", ""))
        agg[name][0] += 1
        agg[name][1] += ns
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':70s} {'launches':>8s} {'total_ms':>10s} {'avg_us':>10s} {'share':>7s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[-70:]:70s} {v[0]:8d} {v[1] / 1e6:10.3f} {v[1] / v[0] / 1e3:10.2f} {v[1] / tot * 100:6.1f}%")
print(f"{'TOTAL':70s} {sum(v[0] for v in agg.values()):8d} {tot / 1e6:10.3f}")

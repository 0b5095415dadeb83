"""Writes profiles/advance_p_ncu.json (read by bench.py for roofline.traffic)
from ncu_summary.py outputs of advance_p launches across a sort cycle.
Usage: make_profile_json.py KERNEL_LABEL summary.txt:STALE [summary.txt:STALE ...]
STALE = steps since the last sort (0 = the push that applies the deferred
permutation).  The per-push traffic is weighted over a 20-step cycle: the
stale-0 launch once, the others sharing the remaining 19 steps equally."""
import json
import os
import sys

label = sys.argv[1]
launches = []
for arg in sys.argv[2:]:
    f, st = arg.rsplit(":", 1)
    line = next(ln for ln in open(f) if ln.startswith("{"))
    d = json.loads(line)
    d["particles"] = 536870912
    d["staleness"] = int(st)
    d["workload"] = "two_stream 256^3, one species launch (2^29 particles)"
    launches.append(d)
g = [d for d in launches if d["staleness"] == 0]
o = [d for d in launches if d["staleness"] != 0]
if g and o:
    per_push = (sum(d["dram_bytes_per_push"] for d in g) / len(g) +
                19 * sum(d["dram_bytes_per_push"] for d in o) / len(o)) / 20
else:
    per_push = sum(d["dram_bytes_per_push"] for d in launches) / len(launches)
out = {"kernel": label, "launches": launches, "dram_bytes_per_push": per_push,
       "dram_bytes_per_launch": per_push * 536870912,
       "note": "ncu --set full --clock-control none, one advance_p launch per staleness; per push = "
               "(dram read + write) / particles, weighted over a 20-step sort cycle (stale 0 = the gathering push "
               "once, the other launches sharing 19 steps)"}
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
json.dump(out, open(os.path.join(root, "profiles", "advance_p_ncu.json"), "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "launches"}))

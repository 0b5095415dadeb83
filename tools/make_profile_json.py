"""Writes profiles/advance_p_ncu.json (read by bench.py for roofline.traffic)
from ncu_summary.py outputs of one fresh and one stale advance_p launch.
Usage: make_profile_json.py KERNEL_LABEL fresh.txt stale.txt [stale_steps]"""
import json
import os
import sys

label, files = sys.argv[1], sys.argv[2:4]
stale = int(sys.argv[4]) if len(sys.argv) > 4 else 19
launches = []
for f, st in zip(files, (0, stale)):
    line = next(ln for ln in open(f) if ln.startswith("{"))
    d = json.loads(line)
    d["particles"] = 536870912
    d["staleness"] = st
    d["workload"] = "two_stream 256^3, one species launch (2^29 particles)"
    launches.append(d)
per_push = sum(d["dram_bytes_per_push"] for d in launches) / len(launches)
out = {"kernel": label, "launches": launches, "dram_bytes_per_push": per_push,
       "dram_bytes_per_launch": per_push * 536870912,
       "note": "ncu --set full --clock-control none, one advance_p launch each (fresh, and "
               f"{stale} steps after a sort); per push = (dram read + write) / particles; mean of the two"}
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
json.dump(out, open(os.path.join(root, "profiles", "advance_p_ncu.json"), "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "launches"}))

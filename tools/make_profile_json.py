"""Writes profiles/advance_p_ncu.json (read by bench.py for roofline.traffic)
from tools/ncu_multi.py JSON lines of consecutive advance_p launches over a
reorder cycle (in-place, counting and reordering pushes of every species).
Usage: make_profile_json.py KERNEL_LABEL PARTICLES_PER_LAUNCH WORKLOAD run.jsonl [OUT_NAME]
(OUT_NAME defaults to advance_p_ncu.json, the headline workload's; bench.py
reads advance_p_ncu_<config>.json for the other configs)
The per-push traffic is the mean over the listed launches (one full cycle:
each launch kind appears as often as it runs)."""
import json
import os
import sys

label, npart, workload, path = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4]
out_name = sys.argv[5] if len(sys.argv) > 5 else "advance_p_ncu.json"
launches = [json.loads(ln) for ln in open(path) if ln.startswith("{")]
for d in launches:
    if d["ms"] > 50 and npart < 1e8:  # older summaries: microseconds in the "ms" field
        d["ms"] /= 1e3
        d["algorithmic_GBs"] *= 1e3
    d["particles"] = npart
per_push = sum(d["dram_bytes_per_push"] for d in launches) / len(launches)
ms = sum(d["ms"] for d in launches) / len(launches)
out = {"kernel": label, "workload": workload, "launches": launches, "dram_bytes_per_push": per_push,
       "dram_bytes_per_launch": per_push * npart, "mean_launch_ms": ms,
       "mean_algorithmic_GBs": npart * 64 / (ms * 1e-3) / 1e9,
       "note": "ncu --set full --clock-control none, consecutive advance_p launches over one reorder cycle "
               "(in-place x3, counting, reordering; one launch pushes every species of the deck; cold caches, "
               "serialised); per push = "
               "(dram read + write) / particles, averaged over the cycle"}
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
json.dump(out, open(os.path.join(root, "profiles", out_name), "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "launches"}))

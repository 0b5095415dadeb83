"""Summarise an ncu --set full report: headline metrics, stall reasons and
per-opcode instruction mix of the profiled kernel.  Usage:
  python tools/ncu_summary.py gpurun_out/prof_X.ncu-rep [n_particles]"""
import collections
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
npart = float(sys.argv[2]) if len(sys.argv) > 2 else None


def page(p, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


raw = page("raw")
hdr, units, vals = raw[0], raw[1], raw[2]
get = {h: (vals[i], units[i]) for i, h in enumerate(hdr)}
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "smsp__inst_executed.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "smsp__inst_executed_op_global_red.sum", "launch__grid_size", "launch__block_size"]
summary = {}
for k in keys:
    if k in get:
        summary[k] = get[k][0] + (" " + get[k][1] if get[k][1] else "")
        print(f"{k:60s} {get[k][0]:>22s} {get[k][1]}")
st = [(h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], float(v or 0))
      for h, (v, u) in get.items() if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
st.sort(key=lambda x: -x[1])
print("stalls per issue:", ", ".join(f"{k}={v:.2f}" for k, v in st[:8]))
summary["stalls_per_issue"] = dict(st[:8])
sass = page("source", ["--print-source=sass"])
h2 = sass[1]
ia, isrc = h2.index("Instructions Executed"), h2.index("Source")
ops = collections.Counter()
tot = 0.0
for r in sass[2:]:
    n = float(r[ia] or 0)
    tot += n
    toks = r[isrc].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    ops[op.split(".")[0]] += n
print("total warp instructions", tot)
if npart:
    print("warp instructions per 32 particles", tot / (npart / 32))
    summary["warp_inst_per_32_particles"] = tot / (npart / 32)
print(", ".join(f"{k}={v / tot * 100:.1f}%" for k, v in ops.most_common(16)))
dram = float(get["dram__bytes_read.sum"][0]) * (1e6 if get["dram__bytes_read.sum"][1] == "Mbyte" else 1e9 if get["dram__bytes_read.sum"][1] == "Gbyte" else 1) + \
    float(get["dram__bytes_write.sum"][0]) * (1e6 if get["dram__bytes_write.sum"][1] == "Mbyte" else 1e9 if get["dram__bytes_write.sum"][1] == "Gbyte" else 1)
summary["dram_bytes"] = dram
if npart:
    summary["dram_bytes_per_push"] = dram / npart
    print("dram bytes per push", dram / npart)
print(json.dumps(summary))

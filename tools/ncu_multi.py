"""Per-launch summary of a multi-launch ncu --set full report of advance_p
(one JSON object per launch: kind from the kOrd template argument, time,
DRAM bytes per push, issue/occupancy, L1/L2 hit rates, top stalls).
Usage: python tools/ncu_multi.py REPORT.ncu-rep PARTICLES_PER_LAUNCH"""
import csv
import io
import json
import subprocess
import sys

rep, npart = sys.argv[1], float(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,
         "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
KIND = {"0": "in-place", "1": "counting", "2": "reordering"}
res = []
for r in rows[2:]:
    g = {h: (r[i], units[i]) for i, h in enumerate(hdr)}

    def num(k):
        v, u = g[k]
        return float(v.replace(",", "")) * SCALE.get(u, 1.0)

    name = g["Kernel Name"][0]
    targs = name[name.find("<") + 1:name.find(">")].split(",")
    # kOrd is the 12th template argument (a 13th, kPk, follows since round 2)
    kind = KIND.get(targs[11 if len(targs) > 12 else -1].strip(), "?") if "advance_p_lean" in name \
        else name.split("(")[0]
    dram = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
    ms = num("gpu__time_duration.sum")
    st = sorted(((h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], float(v[0] or 0))
                 for h, v in g.items() if h.startswith("smsp__average_warps_issue_stalled_")
                 and h.endswith("_per_issue_active.ratio")), key=lambda x: -x[1])[:5]
    d = {"kind": kind, "ms": ms, "dram_bytes": dram, "dram_bytes_per_push": dram / npart,
         "dram_read_per_push": num("dram__bytes_read.sum") / npart,
         "dram_write_per_push": num("dram__bytes_write.sum") / npart,
         "algorithmic_GBs": npart * 64 / (ms * 1e-3) / 1e9,
         "dram_pct_peak": float(g["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"][0]),
         "issue_active_pct": float(g["smsp__issue_active.avg.pct_of_peak_sustained_active"][0]),
         "warps_active_pct": float(g["sm__warps_active.avg.pct_of_peak_sustained_active"][0]),
         "warp_inst_per_32": num("smsp__inst_executed.sum") / (npart / 32),
         "l1_hit_pct": float(g["l1tex__t_sector_hit_rate.pct"][0]),
         "l2_hit_pct": float(g["lts__t_sector_hit_rate.pct"][0]),
         "registers": g["launch__registers_per_thread"][0],
         "stalls_per_issue": dict(st), "kernel": name.split("(")[0]}
    res.append(d)
    print(json.dumps(d))

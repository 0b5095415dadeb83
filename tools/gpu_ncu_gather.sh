#!/bin/bash
# ncu of the gathering push (first push after a deferred sort) vs the next push.
timeout 900 ncu --set full --clock-control none --import-source on -k regex:advance_p_lean -s 40 -c 4 -o gpurun_out/prof_gather \
  python bench.py --steps 2 --warmup 21 --no-e2e --no-cpu-baseline > gpurun_out/ncu_gather.log 2>&1
python - << 'PY'
import subprocess, csv, io
out = subprocess.run(["ncu", "-i", "gpurun_out/prof_gather.ncu-rep", "--page", "raw", "--csv", "--metrics",
                      "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,smsp__average_warp_latency_issue_stalled_long_scoreboard,l1tex__t_sector_hit_rate.pct"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print(d.get("Kernel Name", "")[:60], {k: d[k] for k in hdr if k.startswith(("gpu__", "dram__", "smsp__", "l1tex"))})
PY

#!/bin/bash
# Round-end style measurement pass: GPU suite + smoke, every bench workload,
# the reference arm, launch lists and ncu --set full reorder cycles.
TAG=${1:-fin}
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/gputest_$TAG.txt 2>&1; tail -3 gpurun_out/gputest_$TAG.txt
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/gputest_$TAG.txt 2>&1; tail -1 gpurun_out/gputest_$TAG.txt
timeout 900 python bench.py --steps 20 --warmup 4 > gpurun_out/bench_two_stream_$TAG.json 2> gpurun_out/bench_two_stream_$TAG.err
for C in thermal weak harris lpi; do
  timeout 900 python bench.py --config $C --steps 20 --warmup 4 --no-cpu-baseline > gpurun_out/bench_${C}_$TAG.json 2> gpurun_out/bench_${C}_$TAG.err
done
timeout 900 python bench.py --decomposed --steps 20 --warmup 4 --no-cpu-baseline --no-e2e > gpurun_out/bench_dec_$TAG.json 2> gpurun_out/bench_dec_$TAG.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
for C in two_stream thermal weak harris lpi dec ref; do python - <<PY
import json
try:
    d=json.load(open("gpurun_out/bench_${C}_$TAG.json"))
    r=d.get("roofline") or {}
    print("$C", "%.4g" % d["value"], d.get("ms_per_step"), "frac", r.get("frac"), (d.get("clocks") or {}).get("sm_mhz"), (d.get("clocks") or {}).get("reasons"), "e2e", (d.get("e2e") or {}).get("value"))
except Exception as e:
    print("$C", "ERR", e)
PY
done
for C in thermal two_stream; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_$C.csv \
    python bench.py --config $C --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/l_$C.csv > gpurun_out/launches_${C}_$TAG.txt; gzip -f gpurun_out/l_$C.csv
done
bash tools/gpu_ncu_cycle.sh $TAG
ls gpurun_out

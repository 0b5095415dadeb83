#!/bin/bash
# ncu --set full over one reorder cycle of advance_p launches (batched: one
# launch pushes every species; in place x3, counting, reordering) for the
# thermal C1 and two-stream C2 decks, summarised per launch (ncu_multi) and
# turned into profiles/advance_p_ncu*.json by make_profile_json.
TAG=${1:-cyc}
mkdir -p /tmp/reps
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:advance_p_lean -s 10 -c 5 \
  -o /tmp/reps/th_$TAG python bench.py --config thermal --steps 12 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_multi.py /tmp/reps/th_$TAG.ncu-rep 16777216 > gpurun_out/ncu_thermal_$TAG.jsonl
cut -c1-300 gpurun_out/ncu_thermal_$TAG.jsonl
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:advance_p_lean -s 10 -c 5 \
  -o /tmp/reps/ts_$TAG python bench.py --steps 12 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_multi.py /tmp/reps/ts_$TAG.ncu-rep 1073741824 > gpurun_out/ncu_two_stream_$TAG.jsonl
cut -c1-300 gpurun_out/ncu_two_stream_$TAG.jsonl

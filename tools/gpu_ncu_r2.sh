#!/bin/bash
# ncu --set full over one reorder cycle of advance_p launches (in-place,
# counting and reordering pushes) on the thermal C1 deck (10 launches) and the
# two-stream C2 deck (10 launches = 5 steps x 2 species).
TAG=${1:-r2b}
set -x
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:advance_p_lean -s 20 -c 10 \
  -o /tmp/ncu_thermal_$TAG python bench.py --config thermal --steps 14 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_thermal_$TAG.log 2>&1
python tools/ncu_multi.py /tmp/ncu_thermal_$TAG.ncu-rep 8388608 > gpurun_out/ncu_thermal_$TAG.jsonl
cat gpurun_out/ncu_thermal_$TAG.jsonl | cut -c1-400
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:advance_p_lean -s 20 -c 10 \
  -o /tmp/ncu_two_stream_$TAG python bench.py --steps 14 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_two_stream_$TAG.log 2>&1
python tools/ncu_multi.py /tmp/ncu_two_stream_$TAG.ncu-rep 536870912 > gpurun_out/ncu_two_stream_$TAG.jsonl
cat gpurun_out/ncu_two_stream_$TAG.jsonl | cut -c1-400

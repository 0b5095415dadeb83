#!/bin/bash
# ncu --set full with source of advance_p launches of the thermal deck (one
# reorder cycle), SASS-level stall attribution of the first two (in place).
TAG=${1:-src}
set -x
mkdir -p /tmp/reps
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:advance_p_lean -s 20 -c 10 \
  -o /tmp/reps/th_$TAG python bench.py --config thermal --steps 14 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_th_$TAG.log 2>&1
python tools/ncu_multi.py /tmp/reps/th_$TAG.ncu-rep 8388608 > gpurun_out/ncu_th_$TAG.jsonl
cut -c1-300 gpurun_out/ncu_th_$TAG.jsonl
for k in 0 1 8; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:advance_p_lean -s $((20 + k)) -c 1 \
    -o /tmp/reps/one_${TAG}_$k python bench.py --config thermal --steps 14 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  python tools/ncu_sass_top.py /tmp/reps/one_${TAG}_$k.ncu-rep 80 > gpurun_out/ncu_sass_${TAG}_$k.txt
  ncu -i /tmp/reps/one_${TAG}_$k.ncu-rep --page raw --csv > gpurun_out/ncu_raw_${TAG}_$k.csv
  head -30 gpurun_out/ncu_sass_${TAG}_$k.txt
done

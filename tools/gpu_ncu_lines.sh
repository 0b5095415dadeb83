#!/bin/bash
# Per-source-line and per-SASS stall attribution of single advance_p launches
# of the thermal deck (index k after 20 skipped: 4 = in-place age 3,
# 6 = counting, 8 = reordering electrons).
TAG=${1:-ln}; shift
KS=${@:-4 6 8}
mkdir -p /tmp/reps
for k in $KS; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KRX:-advance_p_lean} -s $((${BASE:-20} + k)) -c 1 \
    -o /tmp/reps/one_${TAG}_$k python bench.py --config thermal --steps 14 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  python tools/ncu_lines.py /tmp/reps/one_${TAG}_$k.ncu-rep 400 > gpurun_out/ncu_lines_${TAG}_$k.txt
  python tools/ncu_sass_top.py /tmp/reps/one_${TAG}_$k.ncu-rep 4000 > gpurun_out/ncu_sass_${TAG}_$k.txt
  python tools/ncu_multi.py /tmp/reps/one_${TAG}_$k.ncu-rep 8388608 > gpurun_out/ncu_one_${TAG}_$k.jsonl
  head -40 gpurun_out/ncu_lines_${TAG}_$k.txt
done

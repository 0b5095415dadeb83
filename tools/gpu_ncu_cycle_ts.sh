#!/bin/bash
# ncu --set full over one reorder cycle of the batched two-stream push (C2).
TAG=${1:-cyc}
mkdir -p /tmp/reps
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:advance_p_lean -s 10 -c 5 \
  -o /tmp/reps/ts_$TAG python bench.py --steps 12 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_multi.py /tmp/reps/ts_$TAG.ncu-rep 1073741824 > gpurun_out/ncu_two_stream_$TAG.jsonl
cut -c1-260 gpurun_out/ncu_two_stream_$TAG.jsonl

#!/bin/bash
# Sort A/B: parity tests, per-variant timings, launch list of the default.
TAG=${1:-s}; VARS=${2:-0,2,3,4}
set -x
timeout 900 python -m pytest tests -m gpu -q -x -k "sort" > gpurun_out/gputest_$TAG.log 2>&1; tail -3 gpurun_out/gputest_$TAG.log
timeout 600 python tools/sort_bench.py two_stream 19 $VARS > gpurun_out/sort_$TAG.txt 2>&1; grep "rep 1" gpurun_out/sort_$TAG.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  -k regex:'radix|scan|count|within|max_kernel|permute' --log-file gpurun_out/sortlaunch_$TAG.csv python tools/sort_bench.py two_stream 19 0 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/sortlaunch_$TAG.csv > gpurun_out/sortlaunch_$TAG.txt; cat gpurun_out/sortlaunch_$TAG.txt

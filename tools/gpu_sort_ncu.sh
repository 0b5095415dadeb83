#!/bin/bash
# Sort kernels: launch list (durations) + ncu --set full of one scatter pass.
TAG=${1:-s1}; VAR=${2:-0}
set -x
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:'radix|scan|count|within|max_kernel' --log-file gpurun_out/sortlaunch_$TAG.csv python tools/sort_bench.py two_stream 19 $VAR > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/sortlaunch_$TAG.csv > gpurun_out/sortlaunch_$TAG.txt; cat gpurun_out/sortlaunch_$TAG.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:radix_scatter -s 2 -c 1 -o gpurun_out/prof_sort_$TAG \
  python tools/sort_bench.py two_stream 19 $VAR > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_sort_$TAG.ncu-rep 536870912 > gpurun_out/prof_sort_$TAG.txt 2>&1; head -30 gpurun_out/prof_sort_$TAG.txt

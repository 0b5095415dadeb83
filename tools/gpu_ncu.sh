#!/bin/bash
# ncu --set full capture of the advance_p kernel on the thermal deck (1 GPU).
set -x
K=${1:-advance_p_kernel}
TAG=${2:-r1}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 8 -c 1 \
  -o gpurun_out/prof_$TAG python bench.py --config thermal --steps 4 --warmup 4 --no-e2e --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1
tail -5 gpurun_out/ncu_$TAG.log
ls -la gpurun_out/

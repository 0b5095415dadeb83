#!/bin/bash
# ncu --set full of one steady-state advance_p launch on the headline C2
# workload, for each PIC_PUSH_VARIANT given (1 GPU; never a bench number).
TAG=$1; shift
for V in "$@"; do
  PIC_PUSH_VARIANT=$V timeout 1200 ncu --set full --clock-control none --import-source on -k regex:advance_p -s 4 -c 1 \
    -o gpurun_out/prof_${TAG}_v$V python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_${TAG}_v$V.log 2>&1
  tail -2 gpurun_out/ncu_${TAG}_v$V.log
done
ls -la gpurun_out/*.ncu-rep

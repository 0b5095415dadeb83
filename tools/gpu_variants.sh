#!/bin/bash
# Push-variant timing table + ncu --set full of chosen variants (1 GPU).
TAG=$1; VARS=$2; NCUVARS=$3
set -x
timeout 1200 python tools/push_variants.py two_stream $VARS 0,10 > gpurun_out/variants_$TAG.txt 2>&1
tail -3 gpurun_out/variants_$TAG.txt
for V in $NCUVARS; do
  PIC_PUSH_VARIANT=$V timeout 1200 ncu --set full --clock-control none --import-source on -k regex:advance_p -s 4 -c 1 \
    -o gpurun_out/prof_${TAG}_v$V python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_${TAG}_v$V.log 2>&1
  tail -2 gpurun_out/ncu_${TAG}_v$V.log
done
ls -la gpurun_out/

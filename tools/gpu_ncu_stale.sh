#!/bin/bash
# ncu --set full of advance_p at a given launch index (staleness) for given
# variants, headline C2 workload.  Usage: TAG "V:SKIP V:SKIP ..."
TAG=$1; shift
for VS in $@; do
  V=${VS%%:*}; SKIP=${VS##*:}
  PIC_PUSH_VARIANT=$V timeout 1200 ncu --set full --clock-control none --import-source on -k regex:advance_p -s $SKIP -c 1 \
    -o gpurun_out/prof_${TAG}_v${V}_s${SKIP} python bench.py --steps 2 --warmup $((SKIP/2+1)) --no-e2e --no-cpu-baseline > gpurun_out/ncu_${TAG}_v${V}_s${SKIP}.log 2>&1
  tail -1 gpurun_out/ncu_${TAG}_v${V}_s${SKIP}.log
done

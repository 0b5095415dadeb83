#!/bin/bash
# ncu --set full of one launch of a kernel (regex) in a bench config, summarised
# on the box (ncu_multi + per-line), report deleted.  Usage: REGEX SKIP CONFIG NPART TAG [env...]
RX=$1; SKIP=$2; CFG=$3; NP=$4; TAG=$5; shift 5
mkdir -p /tmp/reps
env "$@" timeout 900 ncu --set full --clock-control none --import-source on -k regex:$RX -s $SKIP -c 1 \
  -o /tmp/reps/$TAG python bench.py --config $CFG --steps 14 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_multi.py /tmp/reps/$TAG.ncu-rep $NP > gpurun_out/ncu_$TAG.txt
python tools/ncu_lines.py /tmp/reps/$TAG.ncu-rep 400 >> gpurun_out/ncu_$TAG.txt
python tools/ncu_summary.py /tmp/reps/$TAG.ncu-rep $NP | tail -4 >> gpurun_out/ncu_$TAG.txt
head -c 1500 gpurun_out/ncu_$TAG.txt; echo
python tools/ncu_sass_top.py /tmp/reps/$TAG.ncu-rep 60 > gpurun_out/ncu_sass_$TAG.txt

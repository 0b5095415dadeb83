#!/bin/bash
# ncu --set full of one launch of each field kernel (headline deck).
for K in load_interpolators_kernel advance_b_kernel unload_advance_e; do
  timeout 900 ncu --set full --clock-control none -k regex:$K -s 4 -c 1 -o gpurun_out/prof_f_$K \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/prof_f_$K.ncu-rep 17173512 > gpurun_out/prof_f_$K.txt 2>&1
  head -16 gpurun_out/prof_f_$K.txt
done

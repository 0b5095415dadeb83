#!/bin/bash
# Cost decomposition of the ordered push (ablation library, probe variants
# 60-65 = ordered push minus reservation / lidx / counts / per-thread stores)
export PIC_LIB_PATH=$PWD/paper_2102_13133_b200/libpic_b200_ablate.so
for cfg in ${CONFIGS:-weak}; do
  for v in ${VARIANTS:-52 60 61 62 63 64 66}; do
    echo -n "v=$v "; PIC_PUSH_VARIANT=$v python tools/order_probe.py $cfg 4 1
  done
  echo -n "classic "; PIC_PUSH_VARIANT=52 python tools/order_probe.py $cfg 4 0
done

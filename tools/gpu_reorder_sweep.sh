#!/bin/bash
# push-phase rate per step over a sort cycle for reorder intervals m (and the
# in-place push + deferred sort, voxel_order=0), bench decks
for cfg in ${CONFIGS:-weak two_stream thermal}; do
  steps=24
  for m in ${MS:-1 2 3 4 5 6}; do
    echo -n "m=$m "; PIC_REORDER_INTERVAL=$m python tools/order_probe.py $cfg $steps 1
  done
  echo -n "classic "; python tools/order_probe.py $cfg $steps 0
done

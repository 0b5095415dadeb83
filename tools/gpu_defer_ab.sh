#!/bin/bash
# Deferred sort permutation on / off, alternating on one box (whole-step bench).
for D in 1 0 1 0; do
  PIC_SORT_DEFER=$D timeout 900 python bench.py --steps 20 --warmup 4 --no-e2e --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; d=json.load(sys.stdin); print('defer=$D', '%.4g' % d['value'], '%.3f' % d['ms_per_step'], {k: round(v, 3) for k, v in d['config']['phase_ms_per_step'].items()}, d['clocks']['sm_mhz'])"
done

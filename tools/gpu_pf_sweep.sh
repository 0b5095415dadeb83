#!/bin/bash
for E in 0.125 0.1875 0.25 0.375; do
  for C in thermal two_stream; do
    PIC_PF_AHEAD=$E timeout 900 python bench.py --config $C --steps 20 --warmup 4 --no-e2e --no-cpu-baseline 2>/dev/null | \
      python -c "import json,sys; d=json.load(sys.stdin); print('pf=$E', '$C', '%.4g' % d['value'], '%.4f' % d['ms_per_step'], 'kr %.4g' % d['config']['push_kernel_rate'], 'frac', round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"
  done
done

#!/bin/bash
# reorder interval sweep on the batched interleaved push (thermal and two-stream)
for C in thermal two_stream; do
for M in ${MS:-4 5 6 8}; do
  PIC_REORDER_INTERVAL=$M timeout 900 python bench.py --config $C --steps 20 --warmup 4 --no-e2e --no-cpu-baseline 2>/dev/null | \
      python -c "import json,sys; d=json.load(sys.stdin); print('$C m=$M', '%.4g' % d['value'], '%.4f' % d['ms_per_step'], 'kr %.4g' % d['config']['push_kernel_rate'], 'frac', round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"
done; done

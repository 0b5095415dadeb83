#!/bin/bash
# pic_step_host staging depth (PIC_HOST_BUFS) and chunk size A/B: e2e only.
for B in 2 3 4 2 3; do
  PIC_HOST_BUFS=$B timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 2>/dev/null | \
    python -c "import json,sys; d=json.load(sys.stdin); e=d['e2e']; print('bufs=$B', '%.4g' % e['value'], '%.1f ms' % e['ms_per_step'])"
done

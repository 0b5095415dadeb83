#!/bin/bash
# A/B of two library builds (PIC_LIB_PATH) on one box: push variants + whole-step bench.
ALT=$1
for L in default $ALT default $ALT; do
  if [ "$L" = default ]; then unset PIC_LIB_PATH; else export PIC_LIB_PATH=$L; fi
  echo "== $L"
  timeout 600 python tools/push_variants.py two_stream 43 0,19 2>&1 | grep "^stale"
  timeout 900 python bench.py --steps 20 --warmup 4 --no-e2e --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; d=json.load(sys.stdin); print('bench', '%.4g' % d['value'], '%.3f' % d['ms_per_step'], d['clocks']['sm_mhz'])"
done

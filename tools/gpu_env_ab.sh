#!/bin/bash
# Whole-step A/B of an environment setting: bash tools/gpu_env_ab.sh "VAR=a" "VAR=b" [configs]
A=$1; B=$2; CF=${3:-thermal two_stream}
for rep in 1 2; do
for E in "$A" "$B"; do
  for C in $CF; do
    env $E timeout 900 python bench.py --config $C --steps 20 --warmup 4 --no-e2e --no-cpu-baseline 2>/dev/null | \
      python -c "import json,sys; d=json.load(sys.stdin); print('$E', '$C', '%.4g' % d['value'], '%.4f' % d['ms_per_step'], 'frac', round(d['roofline']['frac'],4), 'kr %.4g' % d['config']['push_kernel_rate'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
done

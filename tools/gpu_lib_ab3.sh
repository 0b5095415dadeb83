#!/bin/bash
# Whole-step A/B over several library builds: bash tools/gpu_lib_ab3.sh "default m5 w3m7" [configs]
LIBS=$1; CF=${2:-thermal two_stream}
for rep in 1 2; do
for L in $LIBS; do
  if [ "$L" = default ]; then unset PIC_LIB_PATH; else export PIC_LIB_PATH=$PWD/paper_2102_13133_b200/libpic_b200_$L.so; fi
  for C in $CF; do
    timeout 900 python bench.py --config $C --steps 20 --warmup 4 --no-e2e --no-cpu-baseline 2>/dev/null | \
      python -c "import json,sys; d=json.load(sys.stdin); print('$L', '$C', '%.4g' % d['value'], '%.4f' % d['ms_per_step'], 'frac', round(d['roofline']['frac'],4), 'kr %.4g' % d['config']['push_kernel_rate'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
done
unset PIC_LIB_PATH

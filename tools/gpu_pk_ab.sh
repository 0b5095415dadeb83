#!/bin/bash
# Packed-FP32 push A/B: GPU suite on the packed (default) library, then the
# whole-step bench alternating default / PIC_LIB_PATH=$ALT, and launch lists.
TAG=${1:-pk}; ALT=${2:-$PWD/paper_2102_13133_b200/libpic_b200_scalar.so}
set -x
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_$TAG.txt 2>&1; tail -3 gpurun_out/gputest_$TAG.txt
for rep in 1 2; do
for L in default $ALT; do
  if [ "$L" = default ]; then unset PIC_LIB_PATH; else export PIC_LIB_PATH=$L; fi
  for C in thermal two_stream; do
    timeout 900 python bench.py --config $C --steps 20 --warmup 4 --no-e2e --no-cpu-baseline 2>/dev/null | \
      python -c "import json,sys; d=json.load(sys.stdin); print('$L'[-20:], '$C', '%.4g' % d['value'], '%.4f' % d['ms_per_step'], 'frac', round(d['roofline']['frac'],4), 'kr %.4g' % d['config']['push_kernel_rate'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
done
unset PIC_LIB_PATH
for L in default $ALT; do
  if [ "$L" = default ]; then unset PIC_LIB_PATH; else export PIC_LIB_PATH=$L; fi
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_th.csv \
    python bench.py --config thermal --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/l_th.csv | head -5; rm -f gpurun_out/l_th.csv
done

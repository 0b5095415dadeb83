#!/bin/bash
# order parity; thermal launch lists: default, and the tools library with the
# reordering push's logical indices not moved (timing probe)
TAG=${1:-r2f}
set -x
timeout 900 python -m pytest tests/test_gpu_order.py tests/test_gpu_dd.py -q -x 2>&1 | tail -3
for V in def probe; do
  if [ $V = probe ]; then export PIC_LIB_PATH=$PWD/paper_2102_13133_b200/libpic_b200_ablate.so PIC_ORDER_PROBE=1; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_$V.csv \
    python bench.py --config thermal --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/l_$V.csv | head -8; rm -f gpurun_out/l_$V.csv
done
unset PIC_LIB_PATH PIC_ORDER_PROBE
for C in thermal thermal two_stream; do
  timeout 600 python bench.py --config $C --steps 40 --warmup 4 --no-cpu-baseline --no-e2e > gpurun_out/bench_${C}_$TAG.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bench_${C}_$TAG.json'));print('$C', d['value'], d['ms_per_step'], d['roofline']['frac'], d['config']['push_kernel_rate'], d['clocks']['sm_mhz'])"
done

#!/bin/bash
# order/dd parity + thermal / two-stream bench after a push or order change
TAG=${1:-r2d}
set -x
timeout 900 python -m pytest tests/test_gpu_order.py tests/test_gpu_dd.py tests/test_golden.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3
for C in thermal two_stream thermal; do
  timeout 600 python bench.py --config $C --steps 40 --warmup 4 --no-cpu-baseline --no-e2e > gpurun_out/bench_${C}_$TAG.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bench_${C}_$TAG.json'));print('$C', d['value'], d['ms_per_step'], d['roofline']['frac'], d['config']['push_kernel_rate'], d['clocks']['sm_mhz'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_thermal_$TAG.csv \
  python bench.py --config thermal --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_thermal_$TAG.csv > gpurun_out/launches_thermal_$TAG.txt; head -12 gpurun_out/launches_thermal_$TAG.txt
rm -f gpurun_out/launches_thermal_$TAG.csv

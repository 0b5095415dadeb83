#!/bin/bash
# Relabel A/B + per-line ncu of the thermal pushes (in-place, counting,
# reordering; electrons).  Reports are summarised on the box and deleted.
TAG=${1:-r2c}
set -x
timeout 600 python -m pytest tests/test_gpu_order.py tests/test_golden.py -q -x 2>&1 | tail -3
for RV in 1 0; do
  PIC_RELABEL_VARIANT=$RV timeout 600 python bench.py --config thermal --steps 40 --warmup 4 --no-cpu-baseline --no-e2e > gpurun_out/bench_thermal_rv${RV}_$TAG.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bench_thermal_rv${RV}_$TAG.json'));print('thermal rv$RV', d['value'], d['ms_per_step'], d['roofline']['frac'], d['config']['phase_ms_per_step'])"
done
for RV in 1 0; do
  PIC_RELABEL_VARIANT=$RV timeout 600 python bench.py --steps 20 --warmup 4 --no-cpu-baseline --no-e2e > gpurun_out/bench_ts_rv${RV}_$TAG.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bench_ts_rv${RV}_$TAG.json'));print('two_stream rv$RV', d['value'], d['ms_per_step'], d['roofline']['frac'], d['config']['phase_ms_per_step'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_thermal_$TAG.csv \
  python bench.py --config thermal --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_thermal_$TAG.csv > gpurun_out/launches_thermal_$TAG.txt; head -24 gpurun_out/launches_thermal_$TAG.txt
mkdir -p /tmp/reps
for S in 20 26 28; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:advance_p_lean -s $S -c 1 \
    -o /tmp/reps/th_s$S python bench.py --config thermal --steps 14 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  python tools/ncu_multi.py /tmp/reps/th_s$S.ncu-rep 8388608 > gpurun_out/ncu_th_s${S}_$TAG.txt
  python tools/ncu_lines.py /tmp/reps/th_s$S.ncu-rep 60 >> gpurun_out/ncu_th_s${S}_$TAG.txt
done
python tools/ncu_opdiff.py /tmp/reps/th_s28.ncu-rep /tmp/reps/th_s26.ncu-rep 8388608 > gpurun_out/ncu_opdiff_28_26_$TAG.txt
python tools/ncu_opdiff.py /tmp/reps/th_s26.ncu-rep /tmp/reps/th_s20.ncu-rep 8388608 > gpurun_out/ncu_opdiff_26_20_$TAG.txt
cat gpurun_out/ncu_opdiff_28_26_$TAG.txt

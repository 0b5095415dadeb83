#!/bin/bash
# Round-2 one-GPU pass: GPU tests, smoke, bench lines (headline two-stream,
# thermal C1, weak 256^3), the headline launch list and one ncu --set full of
# the default push.
TAG=${1:-r2a}
set -x
nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_$TAG.log 2>&1; tail -5 gpurun_out/gputest_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -2 gpurun_out/smoke_$TAG.log
for C in two_stream thermal weak; do
  timeout 900 python bench.py --config $C --steps 20 --warmup 4 > gpurun_out/bench_${C}_$TAG.json 2> gpurun_out/bench_${C}_$TAG.err
  cat gpurun_out/bench_${C}_$TAG.json; tail -3 gpurun_out/bench_${C}_$TAG.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; cat gpurun_out/bench_ref_$TAG.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_two_stream_$TAG.csv \
  python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_two_stream_$TAG.csv > gpurun_out/launches_two_stream_$TAG.txt; head -40 gpurun_out/launches_two_stream_$TAG.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_thermal_$TAG.csv \
  python bench.py --config thermal --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_thermal_$TAG.csv > gpurun_out/launches_thermal_$TAG.txt; head -30 gpurun_out/launches_thermal_$TAG.txt
ls gpurun_out

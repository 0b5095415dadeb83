#!/bin/bash
# One-GPU measurement pass: bench lines + ncu launch list of the headline
# workload (numbers printed under ncu are never bench values).
TAG=${1:-r1}
set -x
nproc; free -g | head -2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 900 python bench.py --steps 20 --warmup 4 > gpurun_out/bench_two_stream_$TAG.json 2> gpurun_out/bench_two_stream_$TAG.err
cat gpurun_out/bench_two_stream_$TAG.json; tail -3 gpurun_out/bench_two_stream_$TAG.err
timeout 600 python bench.py --config thermal --steps 20 --warmup 4 --no-cpu-baseline > gpurun_out/bench_thermal_$TAG.json 2> gpurun_out/bench_thermal_$TAG.err
cat gpurun_out/bench_thermal_$TAG.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_two_stream_$TAG.csv \
  python bench.py --steps 20 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_two_stream_$TAG.csv > gpurun_out/launches_two_stream_$TAG.txt
cat gpurun_out/launches_two_stream_$TAG.txt

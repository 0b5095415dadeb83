#!/bin/bash
# One-GPU measurement pass: bench lines + ncu launch list (no numbers from
# under ncu are reported as bench values).
set -x
free -g | head -2; nproc
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 600 python bench.py --config thermal --steps 20 --warmup 4 --no-cpu-baseline > gpurun_out/bench_thermal.json 2> gpurun_out/bench_thermal.err
cat gpurun_out/bench_thermal.json; tail -5 gpurun_out/bench_thermal.err
timeout 1200 python bench.py --steps 20 --warmup 4 > gpurun_out/bench_two_stream.json 2> gpurun_out/bench_two_stream.err
cat gpurun_out/bench_two_stream.json; tail -5 gpurun_out/bench_two_stream.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_thermal.csv python bench.py --config thermal --steps 20 --warmup 4 --no-e2e --no-cpu-baseline > /dev/null 2>&1
tail -3 gpurun_out/launches_thermal.csv

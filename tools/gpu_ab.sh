#!/bin/bash
# A/B pass after a kernel change: GPU tests, sort timings, push variants, bench.
TAG=${1:-ab}; VARS=${2:-30,37,38}
set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_$TAG.log 2>&1; tail -3 gpurun_out/gputest_$TAG.log
timeout 600 python tools/sort_bench.py two_stream 19 0,2 > gpurun_out/sort_$TAG.txt 2>&1; tail -8 gpurun_out/sort_$TAG.txt
timeout 1200 python tools/push_variants.py two_stream $VARS 0,10,19 > gpurun_out/variants_$TAG.txt 2>&1; tail -12 gpurun_out/variants_$TAG.txt
timeout 900 python bench.py --steps 20 --warmup 4 --no-e2e > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json

#!/bin/bash
# Whole-step bench for several push variants (no e2e / cpu arm).
TAG=${1:-bab}; shift
for V in "$@"; do
  PIC_PUSH_VARIANT=$V timeout 900 python bench.py --steps 20 --warmup 4 --no-e2e --no-cpu-baseline > gpurun_out/bench_${TAG}_v$V.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}_v$V.json'));print('v$V', d['value'], d['ms_per_step'], d['config']['phase_ms_per_step'], d['clocks'])"
done

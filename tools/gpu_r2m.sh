#!/bin/bash
# Round-2 re-measurement after the container reset: the full GPU suite, smoke,
# bench lines for every workload, the reference arm, and launch lists.
TAG=${1:-r2m}
set -x
nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/gputest_$TAG.txt 2>&1; tail -25 gpurun_out/gputest_$TAG.txt
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/gputest_$TAG.txt 2>&1; tail -1 gpurun_out/gputest_$TAG.txt
timeout 900 python bench.py --steps 20 --warmup 4 > gpurun_out/bench_two_stream_$TAG.json 2> gpurun_out/bench_two_stream_$TAG.err
cat gpurun_out/bench_two_stream_$TAG.json; tail -3 gpurun_out/bench_two_stream_$TAG.err
for C in thermal weak harris; do
  timeout 900 python bench.py --config $C --steps 20 --warmup 4 --no-cpu-baseline > gpurun_out/bench_${C}_$TAG.json 2> gpurun_out/bench_${C}_$TAG.err
  cut -c1-600 gpurun_out/bench_${C}_$TAG.json; tail -2 gpurun_out/bench_${C}_$TAG.err
done
timeout 900 python bench.py --decomposed --steps 20 --warmup 4 --no-cpu-baseline --no-e2e > gpurun_out/bench_dec_$TAG.json 2> gpurun_out/bench_dec_$TAG.err
cut -c1-600 gpurun_out/bench_dec_$TAG.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
cat gpurun_out/bench_ref_$TAG.json
for C in thermal two_stream; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_$C.csv \
    python bench.py --config $C --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/l_$C.csv > gpurun_out/launches_${C}_$TAG.txt; head -12 gpurun_out/launches_${C}_$TAG.txt
  gzip -f gpurun_out/l_$C.csv
done
ls gpurun_out

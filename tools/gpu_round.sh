#!/bin/bash
# Full one-GPU measurement pass: tests, smoke, bench lines (two-stream headline,
# thermal, decomposed self-exchange), launch list, ncu --set full of the
# default advance_p one step after a sort, 19 steps after, and at the push
# that applies the deferred permutation of the step-20 sort.
TAG=${1:-r1}; V=${2:-52}
set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_$TAG.log 2>&1; tail -3 gpurun_out/gputest_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -2 gpurun_out/smoke_$TAG.log
bash tools/gpu_ncu_stale.sh $TAG $V:2 $V:38 $V:40
for f in gpurun_out/prof_${TAG}_v${V}_s*.ncu-rep; do python tools/ncu_summary.py $f 536870912 > ${f%.ncu-rep}.txt; python tools/ncu_lines.py $f 40 >> ${f%.ncu-rep}.txt; done
python tools/make_profile_json.py "advance_p_lean<8, 6, false, ..., kCQ = true> (push variant $V, default)" \
  gpurun_out/prof_${TAG}_v${V}_s2.txt:1 gpurun_out/prof_${TAG}_v${V}_s38.txt:19 gpurun_out/prof_${TAG}_v${V}_s40.txt:0
cp profiles/advance_p_ncu.json gpurun_out/advance_p_ncu_$TAG.json
bash tools/gpu_bench.sh $TAG > gpurun_out/bench_$TAG.log 2>&1
timeout 900 python bench.py --decomposed --steps 20 --warmup 4 --no-cpu-baseline --no-e2e > gpurun_out/bench_dec_$TAG.json 2> gpurun_out/bench_dec_$TAG.err
ls gpurun_out

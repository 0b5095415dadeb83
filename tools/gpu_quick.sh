#!/bin/bash
# GPU suite + whole-step bench lines for thermal / two-stream / weak.
TAG=${1:-q}
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_$TAG.txt 2>&1; tail -3 gpurun_out/gputest_$TAG.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for C in thermal two_stream weak; do
  timeout 900 python bench.py --config $C --steps 20 --warmup 4 --no-e2e --no-cpu-baseline > gpurun_out/bench_${C}_$TAG.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/bench_${C}_$TAG.json')); print('$C', '%.4g' % d['value'], '%.4f' % d['ms_per_step'], 'frac', round(d['roofline']['frac'],4), 'kr %.4g' % d['config']['push_kernel_rate'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done

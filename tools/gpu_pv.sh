#!/bin/bash
# Push-variant timing tables on the two-stream and thermal decks.
TAG=${1:-pv}; VARS=${2:-30}
set -x
timeout 900 python -m pytest tests -m gpu -q -x -k "advance_p or sort" > gpurun_out/gputest_$TAG.log 2>&1; tail -2 gpurun_out/gputest_$TAG.log
timeout 1200 python tools/push_variants.py two_stream $VARS 0,10,19 > gpurun_out/variants_${TAG}_ts.txt 2>&1; grep "^stale" gpurun_out/variants_${TAG}_ts.txt
timeout 1200 python tools/push_variants.py thermal $VARS 0,10,19 > gpurun_out/variants_${TAG}_th.txt 2>&1; grep "^stale" gpurun_out/variants_${TAG}_th.txt

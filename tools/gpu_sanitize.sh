#!/bin/bash
# compute-sanitizer over tools/sanitize_case.py (every product kernel family),
# one log per tool under gpurun_out/sanitize_<tool>.txt
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 python tools/sanitize_case.py \
    > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$? $(tail -2 gpurun_out/sanitize_$tool.txt | tr '\n' ' ')"
done

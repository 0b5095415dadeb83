# ncu --set full of the deferred sort's first histogram (keys from the records)
# and first / second scatter passes, two-stream 256^3, 19 steps after the load.
TAG=${1:-s3}
mkdir -p gpurun_out
for K in "radix_hist:0:hist1" "radix_scatter:0:scat1" "radix_scatter:1:scat2"; do
  R=${K%%:*}; rest=${K#*:}; S=${rest%%:*}; N=${rest##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${R}" -s $S -c 1 -o gpurun_out/prof_sort_${TAG}_$N \
    python tools/sort_bench.py two_stream 19 0 > gpurun_out/prof_sort_${TAG}_$N.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof_sort_${TAG}_$N.ncu-rep 536870912 > gpurun_out/prof_sort_${TAG}_$N.txt 2>&1
  python tools/ncu_lines.py gpurun_out/prof_sort_${TAG}_$N.ncu-rep 25 >> gpurun_out/prof_sort_${TAG}_$N.txt 2>&1
done

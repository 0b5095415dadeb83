bash tools/gpu_ncu_stale.sh n47 47:38 43:38
for f in gpurun_out/prof_n47_v*_s38.ncu-rep; do python tools/ncu_summary.py $f 536870912 > ${f%.ncu-rep}.txt; python tools/ncu_lines.py $f 30 >> ${f%.ncu-rep}.txt; done

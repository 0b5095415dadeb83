# Sort kernel durations (ncu launch list, two-stream 256^3, 19 steps after the load)
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:'radix|scan' --log-file gpurun_out/sortlaunch_$TAG.csv python tools/sort_bench.py two_stream 19 0 > gpurun_out/sortbench_$TAG.txt 2>&1
python tools/launch_summary.py gpurun_out/sortlaunch_$TAG.csv > gpurun_out/sortlaunch_$TAG.txt
timeout 600 python tools/sort_bench.py two_stream 19 0 > gpurun_out/sortbench_$TAG.txt 2>&1

mkdir -p gpurun_out
timeout 600 python tools/kernel_probe.py two_stream 24 > gpurun_out/kp_loop.txt 2>&1
for cc in all none; do
timeout 900 ncu --kernel-name regex:advance_p_lean --launch-skip 18 --launch-count 2 --cache-control $cc --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum python tools/kernel_probe.py two_stream 11 > gpurun_out/kp_ncu_s10_$cc.txt 2>&1
done
timeout 900 ncu --kernel-name regex:advance_p_lean --launch-skip 40 --launch-count 4 --cache-control all --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum python tools/kernel_probe.py two_stream 22 > gpurun_out/kp_ncu_s21.txt 2>&1

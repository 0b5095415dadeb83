# ncu of the push at stale 19 vs the same physics re-sorted (probe 93 and v52)
mkdir -p gpurun_out
M="--section SpeedOfLight --section WarpStateStats --section MemoryWorkloadAnalysis --section SchedulerStats --section Occupancy --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,smsp__inst_executed_op_global_red.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_read.sum"
for v in 93 52; do
  PIC_SORT_DEFER=0 timeout 900 ncu --kernel-name regex:advance_p_lean --launch-count 1 --clock-control none $M \
    python tools/push_variants.py two_stream $v 19 > gpurun_out/stale_ncu_v${v}.txt 2>&1
  PIC_SORT_DEFER=0 timeout 900 ncu --kernel-name regex:advance_p_lean --launch-count 1 --clock-control none $M \
    python tools/push_variants.py two_stream $v 19 resort > gpurun_out/stale_ncu_v${v}_resort.txt 2>&1
done

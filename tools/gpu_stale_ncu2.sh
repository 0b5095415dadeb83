# ncu of the first push launch at stale 19 for single probes (first launch only: later
# launches see the probes' altered physics)
mkdir -p gpurun_out
for v in 90 91 92 99; do
  timeout 900 ncu --kernel-name regex:advance_p_lean --launch-count 1 --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_red.sum,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio \
    python tools/push_variants.py two_stream $v 19 > gpurun_out/stale_ncu2_v${v}.txt 2>&1
done

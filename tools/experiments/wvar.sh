mkdir -p gpurun_out
for W in 5 9 13 17; do
  BRAX_WARPS_PER_BLOCK=$W python tools/profile_step.py > /dev/null 2>&1 && \
  BRAX_WARPS_PER_BLOCK=$W ncu --section SpeedOfLight --section WarpStateStats --section SchedulerStats --section LaunchStats --section Occupancy --metrics smsp__inst_executed.sum,smsp__pcsamp_warps_issue_stalled_barrier,smsp__pcsamp_warps_issue_stalled_wait --clock-control none -k regex:brax_step -s 3 -c 1 -o gpurun_out/w$W python tools/profile_step.py > gpurun_out/ncu_w$W.log 2>&1
done
python tools/sweep.py --scenes ant --envs 8192 --warps 5,7,9,11,13,17 > gpurun_out/wsweep.log 2>&1

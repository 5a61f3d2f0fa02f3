#!/bin/bash
# Pipe / issue / stall counters of the bench kernel for every library under variants/
# (one k_direct launch each, --clock-control none).  Output: gpurun_out/ncu_variants/<name>.csv
M=sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,smsp__inst_executed.sum,smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_selected_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio
mkdir -p gpurun_out/ncu_variants
for d in variants/*/; do
  n=$(basename $d)
  MCB_LIB=$d/libmcb.so timeout 300 ncu --metrics $M --clock-control none -k regex:k_direct -c 1 --csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-clocks --no-configs \
    > gpurun_out/ncu_variants/$n.csv 2> gpurun_out/ncu_variants/$n.err
done

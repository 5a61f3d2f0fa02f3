#!/usr/bin/env python
"""Summarise an ncu --set full report (every profiled launch): pipe utilisation, issue,
stalls, DRAM traffic.  Usage: tools/ncu_summary.py report.ncu-rep > summary.txt"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration (ms)"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock (GHz)"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid (CTAs)"),
    ("launch__block_size", "CTA size"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("dram__bytes_read.sum", "DRAM read (bytes)"),
    ("dram__bytes_write.sum", "DRAM write (bytes)"),
    ("smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio", "stall: dispatch"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall: math pipe"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall: wait"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall: not selected"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall: short scoreboard"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall: barrier"),
]


def main():
    raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:  # one row per profiled launch
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        print(f"kernel: {d.get('Kernel Name', '?')}")
        for k, label in KEYS:
            if k in d:
                unit = f" {u[k]}" if u.get(k) else ""
                print(f"  {label:28s} {d[k]}{unit}")


if __name__ == "__main__":
    main()

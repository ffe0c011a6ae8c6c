"""Print selected raw metrics of every kernel in an ncu report.

    python tools/ncu_raw.py REPORT.ncu-rep [metric ...]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h, units, rows = r[0], r[1], r[2:]
want = sys.argv[2:] or ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
 'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
 'launch__registers_per_thread', 'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
 'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__grid_size', 'launch__block_size',
 'smsp__inst_executed.sum', 'lts__t_bytes.sum', 'launch__shared_mem_per_block_dynamic',
 'sm__maximum_warps_per_active_cycle_pct',
 'smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio',
 'smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio',
 'smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio',
 'smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio',
 'smsp__issue_active.avg.pct_of_peak_sustained_active', 'l1tex__throughput.avg.pct_of_peak_sustained_active',
 'launch__occupancy_limit_warps', 'sm__ctas_launched.sum']
for vals in rows:
    print("----")
    for i, name in enumerate(h):
        if name in want:
            print(f"{name:80s} {units[i]:16s} {vals[i][:90]}")

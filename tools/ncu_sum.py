"""Key counters of each kernel launch in an ncu report: time, DRAM bytes, instructions, issue/warps active, stalls.
usage: ncu_sum.py REPORT [KERNEL_REGEX]"""
import csv
import io
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
     "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
     "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread", "launch__grid_size",
     "launch__occupancy_limit_registers", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
     "lts__t_bytes.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
     "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
     "smsp__average_warp_latency_issue_stalled_short_scoreboard.ratio",
     "smsp__average_warp_latency_issue_stalled_barrier.ratio",
     "smsp__average_warp_latency_issue_stalled_math_pipe_throttle.ratio",
     "smsp__average_warp_latency_issue_stalled_lg_throttle.ratio",
     "smsp__average_warp_latency_issue_stalled_mio_throttle.ratio",
     "smsp__average_warp_latency_issue_stalled_wait.ratio"]
rep = sys.argv[1]
cmd = ["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(M)]
if len(sys.argv) > 2:
    cmd += ["-k", f"regex:{sys.argv[2]}"]
rows = list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))
h, units = rows[0], rows[1]
for r in rows[2:]:
    print("==", r[h.index("Kernel Name")][:60])
    for m in M:
        if m in h:
            i = h.index(m)
            print(f"   {m:70s} {r[i]:>16s} {units[i]}")

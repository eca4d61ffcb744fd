"""Headline counters of an ncu --set full report (+ the hot-loop opcode mix), for profiles/."""
import csv
import subprocess
import sys

rep, title = sys.argv[1], sys.argv[2]
per = float(sys.argv[3]) if len(sys.argv) > 3 else None
raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                     text=True).stdout.splitlines()))
h, u, v = raw[0], raw[1], raw[2]
print("# " + title)
names = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
         "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
         "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
         "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
         "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed",
         "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
         "lts__t_sector_hit_rate.pct", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
         "launch__shared_mem_per_block_static", "smsp__inst_executed.sum",
         "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
         "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
         "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio"]
for n in names:
    if n in h:
        i = h.index(n)
        print(f"{n:80s} {v[i]} {u[i]}")
if per:
    out = subprocess.run([sys.executable, __file__.replace("ncu_summary.py", "ncu_hot.py"), rep, str(per)],
                         capture_output=True, text=True).stdout.splitlines()
    print("\n".join(l for l in out if l.startswith("instructions") or l.startswith("  ")))

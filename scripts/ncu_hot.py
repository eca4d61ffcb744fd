"""Summarise an ncu --set full report: headline counters + the hot-loop SASS opcode mix."""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
per = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0   # divide counts by this (e.g. #chunks)
raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                     text=True).stdout.splitlines()))
h, v = raw[0], raw[2]
for n in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
          "launch__grid_size", "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
          "dram__throughput.avg.pct_of_peak_sustained_elapsed"):
    if n in h:
        print(f"{n:70s} {v[h.index(n)]}")
src = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                                     capture_output=True, text=True).stdout.splitlines()))
hd = src[1]
ia, isrc = hd.index("Instructions Executed"), hd.index("Source")
ist = hd.index("Warp Stall Sampling (All Samples)")
rows = [(r[isrc], int(r[ia] or 0), int(r[ist] or 0)) for r in src[2:] if len(r) > ia]
tot = sum(r[1] for r in rows)
c, st = Counter(), Counter()
for s, n, smp in rows:
    t = s.split()
    op = t[1] if t and t[0].startswith("@") else (t[0] if t else "?")
    c[op] += n
    st[op] += smp
print(f"instructions executed: {tot}  ({tot / per:.1f} per unit)")
for op, n in c.most_common(30):
    print(f"  {op:22s} {n / per:9.1f}   stall samples {st[op]}")

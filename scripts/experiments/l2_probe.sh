#!/bin/bash
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
run() { echo "== $*"; timeout -s KILL 600 ncu --metrics $M --clock-control none -k regex:logprob_fwd -s 2 -c 1 python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --correction-tokens 0 "$@" 2>&1 | grep -E "duration|dram__|lts__|tensor|cycles_elapsed" | awk '{print $1, $(NF-1), $NF}'; }
run --config c3
run --config c2 --max-pairs 37 --tuning 3,2,1,4,1
run --config c2 --max-pairs 18 --tuning 3,2,1,4,1
run --config c2 --tuning 3,2,1,0,2

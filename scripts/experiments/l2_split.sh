#!/bin/bash
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_requests_evict_first,lts__t_requests_evict_first_lookup_miss,lts__t_requests_evict_last,lts__t_requests_evict_last_lookup_miss,lts__t_sectors_evict_first_lookup_miss,lts__t_sectors_evict_last_lookup_miss,sm__cycles_elapsed.avg.per_second
run() { echo "== $*"; timeout -s KILL 600 ncu --metrics $M --clock-control none -k regex:logprob_fwd -s 2 -c 1 python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --correction-tokens 0 "$@" 2>&1 | grep -E "duration|dram__|lts__|cycles_elapsed" | awk '{print $1, $(NF-1), $NF}'; }
run --config c1 --tuning 3,2,1,4,1
run --config c2 --n-seq 32 --tuning 3,2,1,4,2
run --config c2 --n-seq 32 --tuning 3,2,1,4,8

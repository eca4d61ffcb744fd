#!/bin/bash
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
for t in ${VARIANTS:-3,2,1,4,2 3,2,1,2,2 3,2,1,4,4 3,2,1,2,4 1,2,1,4,2 3,2,1,4,8}; do
  echo "== $t"
  timeout -s KILL 600 ncu --metrics $M --clock-control none -k regex:logprob_fwd -s 2 -c 1 python bench.py --config ${CFG:-c2} --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --correction-tokens 0 --tuning $t 2>&1 | grep -E "duration|dram__|lts__|tensor|cycles_elapsed" | awk '{print $1, $(NF-1), $NF}'
done

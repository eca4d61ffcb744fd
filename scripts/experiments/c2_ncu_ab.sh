#!/bin/bash
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,lts__t_bytes.sum
for t in default 3,1,1,1,4 3,2,1,4,4; do
  if [ "$t" = default ]; then arg=""; else arg="--tuning $t"; fi
  echo "== $t"
  timeout -s KILL 600 ncu --metrics $M --clock-control none -k regex:logprob_fwd -s 3 -c 1 python bench.py --config c2 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --correction-tokens 0 --no-backward-bench --no-sample-bench $arg 2>&1 | grep -E "duration|dram__|lts__|tensor|cycles_elapsed"
done

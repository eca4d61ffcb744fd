#!/bin/bash
# C2-shaped (d = 4096) L2 / DRAM probe matrix on a short batch: group x L2 policies x slack
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second
NSEQ=${NSEQ:-2}
for t in ${VARIANTS:-3,2,1,4,1 3,2,1,4,2 3,2,1,4,4 3,2,1,4,8 1,1,1,4,2 1,1,1,4,4 3,1,1,4,4 1,2,1,4,4 3,2,1,1,4 3,2,1,16,4 3,2,1,0,4 0,0,1,0,2}; do
  echo "== $t"
  timeout -s KILL 300 ncu --metrics $M --clock-control none -k regex:logprob_fwd -s 2 -c 1 python bench.py --config c2 --n-seq $NSEQ --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --correction-tokens 0 --no-sample-bench --no-backward-bench --tuning $t 2>&1 | grep -E "duration|dram__|lts__|cycles_elapsed" | awk '{print $1, $(NF-1), $NF}'
done

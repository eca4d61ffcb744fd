#!/bin/bash
mkdir -p gpurun_out
export PYTHONPATH=$PWD
for t in default 3,2,0,1 3,2,0,2 3,3,0,4 1,2,0,4 3,2,0,2,4; do
timeout -s KILL 300 python scripts/c2_diag.py 2097152 $t 3 >> gpurun_out/c2_diag2.txt 2>&1
done
for t in 3,2,0,1 3,2,0,2; do
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none --csv -k regex:logprob_fwd -c 2 \
   --log-file gpurun_out/c2_ncu_$t.csv python scripts/c2_diag.py 2097152 $t 2 > /dev/null 2>&1
done

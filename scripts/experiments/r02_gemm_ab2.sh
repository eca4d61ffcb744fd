#!/bin/bash
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout -s KILL 400 python scripts/experiments/gemm_knob_ab.py 2048 > gpurun_out/gemm_knob_2048.txt 2>&1
for v in "0 1 1 2 3" "128 1 1 2 3" "128 1 1 1 3" "32 1 1 1 3"; do
set -- $v
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_write.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none --csv -k regex:bwd_gemm \
   --log-file gpurun_out/bwd_ncu_$1_$4.csv python -c "
import sys; sys.argv=['x']
from paper_2605_14220_b200 import tim
tim.debug_set_gemm_slack($1); tim.debug_set_gemm_policy($2,$3,$4,$5)
exec(open('scripts/bwd_once.py').read())
" > /dev/null 2>&1
done

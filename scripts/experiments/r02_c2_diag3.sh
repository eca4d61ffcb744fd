#!/bin/bash
# live-set experiment: DRAM per launch vs the number of live 2-MB H tiles (d = 4096, 524288 tokens)
mkdir -p gpurun_out
export PYTHONPATH=$PWD
M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,lts__t_sector_hit_rate.pct"
run() { # name maxp tuning
  MAXP=$2 timeout -s KILL 600 ncu --metrics $M --clock-control none --csv -k regex:logprob_fwd -c 2 \
   --log-file gpurun_out/c2l_$1.csv python scripts/c2_diag.py 524288 $3 2 > gpurun_out/c2l_$1.txt 2>&1
}
run p74_g2 "" default
run p37_g2 37 default
run p37_g1 37 3,2,0,4,1
run p74_g4 "" 3,2,0,4,4
run p18_g1 18 3,2,0,4,1
run p74_g2_hnorm "" 1,2,0,4

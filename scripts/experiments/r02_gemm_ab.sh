#!/bin/bash
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout -s KILL 300 python scripts/experiments/gemm_slack_ab.py 2048 > gpurun_out/gemm_slack_2048.txt 2>&1
timeout -s KILL 300 python scripts/experiments/gemm_slack_ab.py 4096 > gpurun_out/gemm_slack_4096.txt 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_write.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none --csv -k regex:bwd_gemm \
   --log-file gpurun_out/bwd_launches2.csv python scripts/bwd_once.py --reps 1 > /dev/null 2>&1; echo ncu_rc=$?
timeout -s KILL 300 python -m pytest tests/test_gpu_backward.py -q -x 2>&1 | tail -2

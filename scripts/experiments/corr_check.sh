#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_correct.py -q -x > gpurun_out/tc.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/tc.log
timeout -s KILL 300 python scripts/correct_only.py $((1<<27)); timeout -s KILL 300 python scripts/correct_only.py $((1<<24))
REPS=1 timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed,launch__registers_per_thread -k regex:correct_local -s 0 -c 1 python scripts/correct_only.py > gpurun_out/ncu_corr.txt 2>&1; grep -E "correct_|duration|dram__|fp64|warps_active|issue_active|registers" gpurun_out/ncu_corr.txt | head -30

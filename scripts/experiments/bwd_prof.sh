#!/bin/bash
# head backward: timing split + launch list + ncu of the gradient-epilogue kernel vs the forward kernel
mkdir -p gpurun_out
timeout -s KILL 300 python scripts/bwd_bench.py > gpurun_out/bwd.json 2>&1; echo bwd_rc=$?; tail -1 gpurun_out/bwd.json
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_write.sum,dram__bytes_read.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum --clock-control none --csv \
   --log-file gpurun_out/bwd_launches.csv python scripts/bwd_bench.py > /dev/null 2>&1; echo ncu_rc=$?

#!/bin/bash
# head backward with the tcgen05 GEMMs: timing split vs torch (cuBLAS) matmuls of the same shapes,
# launch list, ncu --set full of the two GEMM kernels
mkdir -p gpurun_out
export PYTHONPATH=$PWD
for d in 2048 4096; do
timeout -s KILL 300 python scripts/bwd_bench.py --d $d > gpurun_out/bwd_$d.json 2>&1; tail -1 gpurun_out/bwd_$d.json
done
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_write.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none --csv \
   --log-file gpurun_out/bwd_launches.csv python scripts/bwd_once.py --reps 2 > /dev/null 2>&1; echo ncu_rc=$?
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:bwd_gemm -c 2 -o gpurun_out/bwd_gemm_full -f python scripts/bwd_once.py > gpurun_out/ncu_full.log 2>&1; echo ncu_full_rc=$?

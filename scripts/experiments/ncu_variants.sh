#!/bin/bash
# dram / L2 / tensor metrics of the logprob kernel per tuning variant (C1)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,lts__t_bytes.sum,l1tex__m_xbar2l1tex_read_bytes.sum
for t in ${VARIANTS:-0,0,0,0 3,2,1,0 3,2,1,4 3,1,1,4 0,0,1,4 3,2,1,16}; do
  timeout -s KILL 600 ncu --metrics $M --clock-control none -k regex:logprob_fwd -s 2 -c 1 --csv \
    python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --tuning $t > gpurun_out/ncuv_$t.csv 2>&1
  echo "== $t"; grep -E '"(gpu__time|dram__bytes|lts__|sm__pipe|sm__cycles|l1tex)' gpurun_out/ncuv_$t.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done

#!/bin/bash
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,l1tex__m_xbar2l1tex_read_bytes.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
run() { echo "== $*"; timeout -s KILL 600 ncu --metrics $M --clock-control none -k regex:logprob_fwd -s 2 -c 1 python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --correction-tokens 0 --no-sample-bench "$@" 2>&1 | grep -E "duration|dram__|lts__|tensor|cycles_elapsed|xbar" | awk '{print $1, $(NF-1), $NF}'; }
run --config c1 --cluster-pairs 1
run --config c1 --cluster-pairs 2
run --config c3 --n-seq 128 --cluster-pairs 1
run --config c3 --n-seq 128 --cluster-pairs 2
for cp in 1 2 1 2; do
  timeout -s KILL 300 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 0 --correction-tokens 0 --no-sample-bench --cluster-pairs $cp > gpurun_out/q_$cp.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/q_$cp.json')); print('bench cluster_pairs=$cp', round(d['value']/1e6,4), 'Mtok/s', round(d['roofline']['achieved'],1), 'TF', d['clocks'])"
done

#!/bin/bash
# tests touching the schedule + bench lines for C1 (default), C2 (d=4096), C3 (8.4M tokens)
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_logprob.py -q -x > gpurun_out/tl.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/tl.log
for c in c1 c2 c3; do
  timeout -s KILL 900 python bench.py --config $c --steps 5 --e2e-steps 2 --cpu-seconds 8 --correction-tokens 0 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c rc=$?
  python -c "import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', round(d['value']/1e6,4), 'Mtok/s', round(d['roofline']['achieved'],1), 'TF', round(d['roofline']['frac_of_burst'],3), d['clocks'], 'e2e', round(d['e2e']['value']/1e6,3))"
done
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
timeout -s KILL 600 ncu --metrics $M --clock-control none -k regex:logprob_fwd -s 2 -c 1 python bench.py --config c2 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --correction-tokens 0 2>&1 | grep -E "duration|dram__|lts__|tensor|cycles_elapsed"

#!/bin/bash
# bench line (C1), ncu --set full of the forward (bench) and of the sampling twin, GPU tests + smoke
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -m gpu -q > gpurun_out/tests_gpu.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/tests_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
timeout -s KILL 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:logprob_fwd -s 2 -c 1 \
   -o gpurun_out/prof_logprob -f python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --correction-tokens 0 --no-sample-bench --no-backward-bench > gpurun_out/ncu_full.log 2>&1; echo ncu_fwd_rc=$?
REPS=1 timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:logprob_fwd -s 2 -c 1 \
   -o gpurun_out/prof_sample -f python scripts/sample_only.py > gpurun_out/ncu_sample.log 2>&1; echo ncu_sample_rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['e2e']['value'], d['sample_twin']['tokens_per_s'], d['head_backward']['tokens_per_s'], d['head_backward']['saved']['tokens_per_s'], d['clocks'])"

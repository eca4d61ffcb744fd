for rep in 1 2 3; do
for lib in libtim_old libtim; do
  L=$PWD/paper_2605_14220_b200/$lib.so
  TIM_LIBRARY=$L timeout -s KILL 300 python scripts/sample_only.py | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read().strip()); print('$rep $lib sample', round(d['tokens_per_s']/1e6,4), d['ids_sum'])"
  TIM_LIBRARY=$L timeout -s KILL 600 python bench.py --steps 10 --no-cpu-baseline --e2e-steps 0 --correction-tokens 0 --no-backward-bench --no-sample-bench > gpurun_out/m.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/m.json')); print('$rep $lib c1', round(d['value']/1e6,4), d['clocks']['sm_mhz'])"
done
done

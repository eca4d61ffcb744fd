#!/bin/bash
# Round 2 (late): host-input path, the kernels on the library's own stream with each copy one chunk
# ahead (new) vs every copy enqueued first and the kernels on the caller's stream (v1); C2 bench
# e2e, interleaved; then the host-path bitwise test.
mkdir -p gpurun_out
for rep in 1 2; do
for v in new v1; do
  if [ $v = v1 ]; then export TIM_HOST_V1=1; else unset TIM_HOST_V1; fi
  timeout -s KILL 900 python bench.py --steps 3 --e2e-steps 3 --no-extra-configs --no-backward-bench --no-sample-bench --correction-tokens 0 --no-cpu-baseline > gpurun_out/e2e_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/e2e_$v.json')); print('$rep $v value', round(d['value']/1e6,4), 'e2e', round(d['e2e']['value']/1e6,4), 'e2e ms/step', round(d['e2e']['ms_per_step'],1), 'dev ms/step', round(d['ms_per_step'],1))"
done
done
unset TIM_HOST_V1
python -m pytest tests/test_gpu_logprob.py -m gpu -q -k host 2>&1 | tail -1

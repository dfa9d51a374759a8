#!/bin/bash
# SGD kernel time from bench.py under several environment settings: bash tools/bench_sgd_only.sh "ENV=.. ENV2=.." ...
for cfg in "$@"; do
  env $cfg timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$cfg', 'step', round(d['ms_per_step'],2), 'sgd', round(d['kernels']['sgd_kernel']['ms_per_step'],3), 'clk', d['clocks']['sm_mhz'])"
done

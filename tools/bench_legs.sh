#!/bin/bash
# C4/C5 scaling-leg times from bench.py under several environment settings
for cfg in "$@"; do
  env $cfg timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); L=d['scaling_legs']
print('$cfg', 'C4 ms', round(L['C4_sharded_knn']['ms'],1), L['C4_sharded_knn']['sha1'], 'C5 ms', round(L['C5_distributed_inference']['ms'],1), L['C5_distributed_inference']['sha1'], 'transform_sgd', round(d['kernels'].get('transform_sgd_kernel',{}).get('ms_per_step',0),2))"
done

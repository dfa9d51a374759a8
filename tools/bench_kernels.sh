#!/bin/bash
# per-kernel ms from bench.py under several environment settings
for cfg in "$@"; do
  env $cfg timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-scaling-legs 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); K=d['kernels']
print('$cfg', 'step', round(d['ms_per_step'],2), 'fine', round(K['knn_tc_kernel (trust ranks)']['ms_per_step'],2), 'coarse', round(K['knn_tc_kernel (trust coarse)']['ms_per_step'],2), 'rank_fix', round(K['rank_fix_kernel']['ms_per_step'],2), 'sgd', round(K['sgd_kernel']['ms_per_step'],2), 'frac_fine', round(d['trust_fine_tile_fraction'],3), 'T', d['trustworthiness'], 'amb', d['trust_ambiguous_pairs'], 'clk', d['clocks']['sm_mhz'])"
done

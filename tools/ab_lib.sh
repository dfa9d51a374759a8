# same-box A/B of alternate libraries: bash tools/ab_lib.sh name...  (tools/_alt_<name>.so)
for v in "$@" "$@"; do
  cp tools/_alt_$v.so paper_2008_00325_b200/libumapb200.so
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-scaling-legs --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('ab $v', round(d['ms_per_step'],3), 'T', d['trustworthiness'], {k: round(v,3) for k,v in d['stages_ms'].items()}, {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items() if 'trust' in k})"
done

#!/bin/bash
# Fine-pass chunk order A/B on one box (bench C2 step + ncu DRAM bytes of the tensor kernels per variant).
# usage (on the GPU box): bash tools/ab_fine.sh "TMAJ CH" ...
mkdir -p gpurun_out
for v in "$@"; do
  set -- $v
  for rep in 1 2; do
    UMAP_TC_TILE_MAJOR=$1 UMAP_TC_CHUNK=$2 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-scaling-legs --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('ab tmaj=$1 ch=$2', round(d['ms_per_step'],3), 'T', d['trustworthiness'], {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items() if 'knn_tc' in k})"
  done
  UMAP_TC_TILE_MAJOR=$1 UMAP_TC_CHUNK=$2 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum \
     --clock-control none -k regex:knn_tc --csv --log-file gpurun_out/ab_ncu_$1_$2.csv \
     python tools/profile_step.py --knn-mode tensor > /dev/null 2>&1
done

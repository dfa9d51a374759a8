#!/bin/bash
# ncu --set full of the deterministic SGD kernel at C2 (one launch), with the SASS source page.
# usage: bash tools/ncu_sgd.sh <tag> [kernel regex]
TAG=${1:-x}; KR=${2:-sgd_flat2}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KR" -c 1 -o /tmp/sgd_${TAG} -f \
    python tools/profile_step.py --knn-mode tensor --no-trust > gpurun_out/ncu_sgd_${TAG}.log 2>&1
ncu -i /tmp/sgd_${TAG}.ncu-rep --page details > gpurun_out/ncu_sgd_${TAG}_details.txt 2>/dev/null
ncu -i /tmp/sgd_${TAG}.ncu-rep --page raw --csv --print-units base > gpurun_out/ncu_sgd_${TAG}_raw.csv 2>/dev/null
ncu -i /tmp/sgd_${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_sgd_${TAG}_sass.csv 2>/dev/null
gzip -f gpurun_out/ncu_sgd_${TAG}_sass.csv gpurun_out/ncu_sgd_${TAG}_raw.csv
tail -3 gpurun_out/ncu_sgd_${TAG}.log
grep -E "Duration|Issue Slots|Eligible Warps|L2 Cache Throughput|L1/TEX Hit|Executed Instructions  |No Eligible" gpurun_out/ncu_sgd_${TAG}_details.txt | head -12

#!/bin/bash
# ncu --set full of the kNN tensor kernel (MODE 0) alone, SASS-level source page exported.
TAG=${1:-knn}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:knn_tc -c 1 -o /tmp/prof_${TAG} -f \
    python tools/tc_debug_time.py > gpurun_out/prof_${TAG}.log 2>&1
ncu -i /tmp/prof_${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${TAG}_sass.csv 2>/dev/null
ncu -i /tmp/prof_${TAG}.ncu-rep --page details > gpurun_out/prof_${TAG}_details.txt 2>/dev/null
gzip -f gpurun_out/prof_${TAG}_sass.csv
ls -la gpurun_out | grep ${TAG}

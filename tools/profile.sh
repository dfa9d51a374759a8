#!/bin/bash
# usage (on the GPU box): bash tools/profile.sh <tag> [extra args for profile_step.py]
# 1) launch list of one step; 2) ncu --set full of the main kernels.
set -x
TAG=$1; shift
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python tools/profile_step.py "$@" > gpurun_out/launches_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'dist_tile|sgd_epoch|union_rows|sort_t_rows|scatter_t|smooth_knn|thresholds|knn_tc' \
    -c 8 -o gpurun_out/prof_${TAG} -f python tools/profile_step.py "$@" > gpurun_out/prof_${TAG}.log 2>&1
ls -la gpurun_out

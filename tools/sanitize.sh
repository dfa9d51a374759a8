#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over tools/sanitize_run.py, with
# every SGD kernel variant.  usage: bash tools/sanitize.sh <tag>
TAG=${1:-r02}
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for var in 0 101 100; do
    log=gpurun_out/sanitize_${TAG}_${tool}_v${var}.log
    UMAP_SGD_VARIANT=$var timeout 1500 $CS --tool $tool --kernel-name-exclude kns=at::,kns=void\ at:: \
        --print-limit 20 python tools/sanitize_run.py > $log 2>&1
    echo "$tool variant=$var rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $log | tail -1) $(grep -c '^ok' $log)"
  done
done

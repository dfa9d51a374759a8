#!/bin/bash
# SGD iteration on the GPU box: SGD parity tests, launch-shape bit-identity, bench (kernel split).
# usage: bash tools/gpu_sgd_iter.sh <tag> [pytest -k expr]
TAG=${1:-x}; K=${2:-"(sgd or optimize or fit or hogwild) and not c2_full"}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "$K" 2>&1 | tail -5 > gpurun_out/pytest_sgd_${TAG}.log
for vt in 0 256 700; do
  if [ $vt = 0 ]; then timeout 300 python tools/sgd_same.py; else UMAP_SGD_VT=$vt timeout 300 python tools/sgd_same.py; fi
done > gpurun_out/sgd_same_${TAG}.log 2>&1
UMAP_SGD_VARIANT=101 timeout 300 python tools/sgd_same.py >> gpurun_out/sgd_same_${TAG}.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
UMAP_SGD_VARIANT=101 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_old.json 2>> gpurun_out/bench_${TAG}.err
cat gpurun_out/pytest_sgd_${TAG}.log gpurun_out/sgd_same_${TAG}.log
for f in gpurun_out/bench_${TAG}.json gpurun_out/bench_${TAG}_old.json; do
python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], "step", round(d["ms_per_step"],2), "sgd", round(d["kernels"]["sgd_kernel"]["ms_per_step"],3), "T", d["trustworthiness"], "clk", d["clocks"]["sm_mhz"])
except Exception as e: print(sys.argv[1], "ERR", e)
PY
done

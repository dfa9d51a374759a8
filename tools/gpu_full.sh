#!/bin/bash
# One GPU call: parity tests, smoke, bench, launch list + ncu --set full of the top kernels.
# usage (on the GPU box): bash tools/gpu_full.sh <tag>
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_${TAG}.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 600 python bench.py --sgd-mode hogwild --no-cpu-baseline --no-e2e > gpurun_out/bench_hog_${TAG}.json 2>> gpurun_out/bench_${TAG}.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-scaling-legs > gpurun_out/launches_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'knn_tc|sgd_|rerank|rank_fix' \
    -c 6 -o /tmp/prof_${TAG} -f python tools/profile_step.py --knn-mode tensor > gpurun_out/prof_${TAG}.log 2>&1
ncu -i /tmp/prof_${TAG}.ncu-rep --page raw --csv --print-units base > gpurun_out/prof_${TAG}_raw.csv 2>/dev/null
ncu -i /tmp/prof_${TAG}.ncu-rep --page details > gpurun_out/prof_${TAG}_details.txt 2>/dev/null
ncu -i /tmp/prof_${TAG}.ncu-rep --page source --csv --print-source sass -k regex:knn_tc --launch-skip 2 --launch-count 1 > gpurun_out/prof_${TAG}_trust_sass.csv 2>/dev/null
ncu -i /tmp/prof_${TAG}.ncu-rep --page source --csv --print-source sass -k regex:sgd_ > gpurun_out/prof_${TAG}_sgd_sass.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/prof_${TAG}_raw.csv gpurun_out/ncu_${TAG}.json > gpurun_out/ncu_${TAG}_summary.txt 2>&1
python tools/launches.py gpurun_out/launches_${TAG}.csv > gpurun_out/launches_${TAG}.txt 2>&1
gzip -f gpurun_out/prof_${TAG}_*sass.csv gpurun_out/prof_${TAG}_raw.csv
du -sh gpurun_out
ls -la gpurun_out
tail -n 3 gpurun_out/pytest_gpu_${TAG}.log gpurun_out/smoke_${TAG}.log
cat gpurun_out/bench_${TAG}.json gpurun_out/bench_hog_${TAG}.json

#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_e2e.py -m gpu -q -k "not c2_full" 2>&1 | tail -8 > gpurun_out/pytest_e2e_r02c.log
timeout 900 python bench.py > gpurun_out/bench_r02c.json 2> gpurun_out/bench_r02c.err
UMAP_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --no-e2e > gpurun_out/bench_r02c_n2.json 2> gpurun_out/bench_r02c_n2.err
cat gpurun_out/pytest_e2e_r02c.log
python - <<'PY'
import json
for f in ["gpurun_out/bench_r02c.json", "gpurun_out/bench_r02c_n2.json"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, "step", d["ms_per_step"], "sgd", d["kernels"].get("sgd_kernel", {}).get("ms_per_step"), "T", d["trustworthiness"])
        print(" legs", json.dumps(d.get("scaling_legs")))
        print(" cpu", json.dumps(d.get("cpu_baseline"))[:600])
    except Exception as e:
        print(f, "ERR", e)
PY
tail -5 gpurun_out/bench_r02c.err gpurun_out/bench_r02c_n2.err

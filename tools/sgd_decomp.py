"""SGD timing decomposition at C2: build the graph once, then time umap_optimize (500 epochs,
deterministic) under UMAP_SGD_DEBUG variants (results are wrong by construction for every
variant but 0; measurement only).  Also hashes Y of the default run (bit-identity checks across
kernel changes).

    python tools/sgd_decomp.py [variants ...]     (default: 0 2 4 12 16 28)
"""
import hashlib
import json
import os
import sys

os.environ.setdefault("UMAP_UNSAFE_EXPERIMENTS", "1")  # this tool reads measurement-only knobs
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2008_00325_b200 as U  # noqa: E402

c = synth.CONFIGS["C2"]
X = torch.from_numpy(synth.lowrank(c["n"], c["d"], c["blobs"], c["seed"])).cuda()
idx, dist = U.knn(X, X, 15, exclude_self=True, mode="tensor")
rho, sigma, w, cs = U.smooth_knn(dist, idx, sort_by_col=True)
indptr, col, val = U.fuzzy_union(cs, w)
a, b = U.fit_ab(0.1, 1.0)
variants = [int(v) for v in sys.argv[1:]] or [0, 2, 4, 12, 16, 28]
Y0 = U.random_init(X.shape[0], 2, 1)
for v in variants:
    os.environ["UMAP_SGD_DEBUG"] = str(v)
    ts = []
    for rep in range(4):
        Y = Y0.clone()
        torch.cuda.synchronize()
        U.profile_begin()
        pos = U.optimize(indptr, col, val, Y, 1, 500, n_epochs=500, a=a, b=b, seed=1, sgd_mode="deterministic")
        p = U.profile_end()
        ts.append(p["sgd_kernel"][0])
        sch = p.get("sgd schedule (count + fill)", (0.0, 0))[0]
    h = hashlib.sha1(Y.cpu().numpy().tobytes()).hexdigest()[:16]
    print(json.dumps({"debug": v, "sgd_ms": [round(t, 3) for t in ts[1:]], "sched_ms": round(sch, 3), "positives": pos, "sha1": h,
                      "sched_mode": os.environ.get("UMAP_SGD_SCHED", "2")}), flush=True)
os.environ.pop("UMAP_SGD_DEBUG", None)

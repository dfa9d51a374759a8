"""End-to-end trust of C1 fits over several seeds at a given n_components, GPU (both SGD modes)
and, with --oracle, the CPU oracle (deterministic): separates chaotic trajectory divergence
from a systematic difference.   python tools/dim_trust_seeds.py DIM [--oracle]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402

A_, B_ = 1.5769434603, 0.8950608779
dim = int(sys.argv[1])
seeds = range(6)
X = synth.make("C1")
if "--oracle" in sys.argv:
    from oracle import oracle as O
    for s in seeds:
        Y = O.fit(X, k=15, n_components=dim, n_epochs=200, a=A_, b=B_, seed=s, mode="deterministic")
        print(json.dumps({"who": "oracle", "dim": dim, "seed": s, "T": O.trustworthiness(X, Y, 15)}), flush=True)
else:
    import torch
    import paper_2008_00325_b200 as U
    Xg = torch.from_numpy(X).cuda()
    for s in seeds:
        for mode in ("deterministic", "hogwild"):
            Y, _ = U.fit(Xg, n_neighbors=15, n_components=dim, n_epochs=200, a=A_, b=B_, seed=s, sgd_mode=mode)
            T, _ = U.trustworthiness(Xg, Y, 15)
            print(json.dumps({"who": "gpu", "mode": mode, "dim": dim, "seed": s, "T": T}), flush=True)

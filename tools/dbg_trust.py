import os, sys
sys.path.insert(0, "/root/repo")
import torch, synth, numpy as np
import paper_2008_00325_b200 as U
c = synth.CONFIGS["C2"]
X = torch.from_numpy(synth.lowrank(c["n"], c["d"], c["blobs"], c["seed"])).cuda()
for seed in [0, 1]:
    Y, st = U.fit(X, n_neighbors=15, n_epochs=500, knn_mode="tensor", seed=seed)
    Yh = Y.cpu().numpy()
    print("seed", seed, "Y finite", np.isfinite(Yh).all(), Yh.min(0), Yh.max(0), flush=True)
    ei, ed = U.knn(Y, Y, 15, exclude_self=True)
    ein = ei.cpu().numpy()
    print("emb idx min/max", ein.min(), ein.max(), flush=True)
    try:
        T, S = U.trustworthiness(X, Y, 15, knn_mode="exact")
        print("exact", T, S, flush=True)
    except Exception as e:
        print("exact failed", e, flush=True)
    T, S = U.trustworthiness(X, Y, 15, knn_mode="tensor")
    print("tensor", T, S, flush=True)

"""C4-shaped (1M x 50) tensor kNN kernel time with and without the short-K prefilter (UMAP_TC_PREFILTER)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, synth
import paper_2008_00325_b200 as U
X = torch.from_numpy(synth.lowrank(1000000, 50, 30, 3)).cuda()
for pf in ["1", "0", "1"]:
    os.environ["UMAP_TC_PREFILTER"] = pf
    U.knn(X, X, 15, exclude_self=True, mode="tensor"); torch.cuda.synchronize()
    U.profile_begin(); i1, d1 = U.knn(X, X, 15, exclude_self=True, mode="tensor"); p = U.profile_end()
    print(pf, {k: round(v[0], 2) for k, v in p.items()}, int(i1[12345, 0]), flush=True)

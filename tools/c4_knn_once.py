"""One C4-shaped (1M x 50) tensor kNN call (for ncu captures of the short-K kernel)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2008_00325_b200 as U
X = torch.from_numpy(synth.lowrank(1000000, 50, 30, 3)).cuda()
i1, d1 = U.knn(X, X, 15, exclude_self=True, mode="tensor")
torch.cuda.synchronize()
print("ok", int(i1[12345, 0]))

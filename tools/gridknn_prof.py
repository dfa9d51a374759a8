import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2008_00325_b200 as U
c = synth.CONFIGS["C2"]
X = torch.from_numpy(synth.lowrank(c["n"], c["d"], c["blobs"], c["seed"])).cuda()
Y, st = U.fit(X, n_neighbors=15, n_epochs=500, knn_mode="tensor")
for i in range(3):
    U.profile_begin()
    gi, gd = U.knn(Y, Y, 15, exclude_self=True)
    p = U.profile_end()
print(os.environ.get("UMAP_GRID_PPC", "4"), {k: round(v[0], 3) for k, v in p.items()})

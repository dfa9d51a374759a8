import os, sys
os.environ.setdefault("UMAP_UNSAFE_EXPERIMENTS", "1")  # this tool reads measurement-only knobs
sys.path.insert(0, "/root/repo")
import torch, synth
import paper_2008_00325_b200 as U
c = synth.CONFIGS["C2"]
X = torch.from_numpy(synth.lowrank(c["n"], c["d"], c["blobs"], c["seed"])).cuda()
for i in range(3):
    U.profile_begin()
    Y, st = U.fit(X, n_neighbors=15, n_epochs=500, knn_mode="tensor")
    p = U.profile_end()
print(os.environ.get("UMAP_SGD_VARIANT", "0"), "ms_sgd", round(st["ms_sgd"], 2), "kernel", round(p["sgd_kernel"][0], 2))

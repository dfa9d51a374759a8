"""Measurement only: kNN / trust tensor-kernel time with parts disabled (UMAP_TC_DEBUG bit0 =
no epilogue filtering, bit1 = no MMA issue) to see which part bounds the kernel."""
import os, sys
os.environ.setdefault("UMAP_UNSAFE_EXPERIMENTS", "1")  # this tool reads measurement-only knobs
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2008_00325_b200 as U
c = synth.CONFIGS["C2"]
X = torch.from_numpy(synth.lowrank(c["n"], c["d"], c["blobs"], c["seed"])).cuda()
for i in range(3):
    U.profile_begin()
    U.knn(X, X, 15, exclude_self=True, mode="tensor")
    p = U.profile_end()
print(os.environ.get("UMAP_TC_DEBUG", "0"), {k: round(v[0], 3) for k, v in p.items()})
Y, st = U.fit(X, n_neighbors=15, n_epochs=500, knn_mode="tensor")
for i in range(2):
    U.profile_begin()
    U.trustworthiness(X, Y, 15, knn_mode="tensor")
    p = U.profile_end()
print("trust", os.environ.get("UMAP_TC_DEBUG", "0"), {k: round(v[0], 3) for k, v in p.items()})

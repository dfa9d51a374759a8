"""Deterministic SGD: hash of Y after a C2 fit (compare across UMAP_SGD_VARIANT values)."""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2008_00325_b200 as U
c = synth.CONFIGS["C2"]
X = torch.from_numpy(synth.lowrank(c["n"], c["d"], c["blobs"], c["seed"])).cuda()
Y, st = U.fit(X, n_neighbors=15, n_epochs=500, knn_mode="tensor", sgd_mode="deterministic")
print(f"variant={os.environ.get('UMAP_SGD_VARIANT', '0')} Y sha1={hashlib.sha1(Y.cpu().numpy().tobytes()).hexdigest()[:16]} positives={st.get('positives')}")

"""SGD launch-shape sweep at C2 (UMAP_SGD_VARIANT read once per process): ms_sgd of 3 fits."""
import os, sys
os.environ.setdefault("UMAP_UNSAFE_EXPERIMENTS", "1")  # this tool reads measurement-only knobs
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2008_00325_b200 as U
c = synth.CONFIGS["C2"]
X = torch.from_numpy(synth.lowrank(c["n"], c["d"], c["blobs"], c["seed"])).cuda()
mode = sys.argv[1] if len(sys.argv) > 1 else "deterministic"
t = []
for i in range(4):
    Y, st = U.fit(X, n_neighbors=15, n_epochs=500, knn_mode="tensor", sgd_mode=mode)
    t.append(st["ms_sgd"])
print(f"variant={os.environ.get('UMAP_SGD_VARIANT', '0')} {mode} ms_sgd={[round(x, 2) for x in t[1:]]}", flush=True)

"""Measurement for planning (results of the overridden margins are NOT certified): ambiguous
pairs and rank_fix time at the certified fine margin and at 1e-4 / 7e-5 (what a separate
lo-product accumulator would allow)."""
import os, sys
os.environ.setdefault("UMAP_UNSAFE_EXPERIMENTS", "1")  # this tool reads measurement-only knobs
sys.path.insert(0, os.getcwd())
import torch, synth
import paper_2008_00325_b200 as U
c = synth.CONFIGS["C2"]
X = torch.from_numpy(synth.lowrank(c["n"], c["d"], c["blobs"], c["seed"])).cuda()
Y, st = U.fit(X, n_neighbors=15, n_epochs=500, knn_mode="tensor")
for m in [None, "1.0e-4", "7e-5"]:
    if m: os.environ["UMAP_TRUST_MARGIN_EXPERIMENT"] = m
    for i in range(2):
        U.profile_begin(); T, S = U.trustworthiness(X, Y, 15, knn_mode="tensor"); p = U.profile_end()
    print(m, U.trust_ambiguous_count(), S, {k: round(v[0], 3) for k, v in p.items() if "rank" in k}, flush=True)

"""Measurement: ambiguous pairs, penalty and rank_fix time with R2's error taken relative to d2
(default) vs folded into the S margin (UMAP_TC_R2_IN_MARGIN, the round-1 form), C2 shape."""
import os, sys
os.environ.setdefault("UMAP_UNSAFE_EXPERIMENTS", "1")  # this tool reads measurement-only knobs
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2008_00325_b200 as U
c = synth.CONFIGS["C2"]
X = torch.from_numpy(synth.lowrank(c["n"], c["d"], c["blobs"], c["seed"])).cuda()
Y, st = U.fit(X, n_neighbors=15, n_epochs=500, knn_mode="tensor")
for mode in ["relative", "in_margin", "relative"]:
    if mode == "in_margin":
        os.environ["UMAP_TC_R2_IN_MARGIN"] = "1"
    else:
        os.environ.pop("UMAP_TC_R2_IN_MARGIN", None)
    for i in range(3):
        U.profile_begin()
        T, S = U.trustworthiness(X, Y, 15, knn_mode="tensor")
        prof = U.profile_end()
    print(f"{mode}: ambiguous {U.trust_ambiguous_count()} S {S} "
          + " ".join(f"{k}={v[0]:.3f}" for k, v in prof.items()), flush=True)

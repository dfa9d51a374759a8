"""Measurement only: ambiguous-pair count and trust time of the tensor-mode penalty vs the
certification margin c (env UMAP_TRUST_MARGIN_EXPERIMENT) at C2 shape."""
import os, sys, time
os.environ.setdefault("UMAP_UNSAFE_EXPERIMENTS", "1")  # this tool reads measurement-only knobs
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2008_00325_b200 as U
c = synth.CONFIGS["C2"]
X = torch.from_numpy(synth.lowrank(c["n"], c["d"], c["blobs"], c["seed"])).cuda()
Y, st = U.fit(X, n_neighbors=15, n_epochs=500, knn_mode="tensor")
T0, S0 = U.trustworthiness(X, Y, 15, knn_mode="tensor")
for m in ["5e-4", "2.5e-4", "1e-4", "5e-5", "2.5e-5", "1e-5"]:
    os.environ["UMAP_TRUST_MARGIN_EXPERIMENT"] = m
    U.trustworthiness(X, Y, 15, knn_mode="tensor")
    torch.cuda.synchronize(); t = time.perf_counter()
    T, S = U.trustworthiness(X, Y, 15, knn_mode="tensor")
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"margin {m}: ambiguous {U.trust_ambiguous_count()} ({U.trust_ambiguous_count() / c['n']:.1f}/row) "
          f"S {S} (ref {S0}, diff {S - S0}) time {dt * 1e3:.1f} ms", flush=True)

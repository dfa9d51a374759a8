"""One C2 step (fit + trust) for ncu: python tools/profile_step.py [--knn-mode exact|tensor] [--sgd-mode ...]"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_2008_00325_b200 as U

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--knn-mode", default="exact")
ap.add_argument("--sgd-mode", default="deterministic")
ap.add_argument("--no-trust", action="store_true")
ap.add_argument("--epochs", type=int, default=0)
a = ap.parse_args()
c = synth.CONFIGS[a.config]
X = torch.from_numpy(synth.lowrank(c["n"], c["d"], c["blobs"], c["seed"])).cuda()
Y, st = U.fit(X, n_neighbors=c["k"], n_epochs=a.epochs or c["n_epochs"], knn_mode=a.knn_mode, sgd_mode=a.sgd_mode)
print(st)
if not a.no_trust:
    print(U.trustworthiness(X, Y, 15, knn_mode=a.knn_mode))

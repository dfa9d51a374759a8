"""Measurement only: how the input-space rank buckets of trustworthiness (R16) are populated
at C2 (which bucket the columns below each row's largest threshold fall into)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2008_00325_b200 as U
c = synth.CONFIGS["C2"]
X = torch.from_numpy(synth.lowrank(c["n"], c["d"], c["blobs"], c["seed"])).cuda()
Y, st = U.fit(X, n_neighbors=15, n_epochs=500, knn_mode="tensor")
ei, _ = U.knn(Y, Y, 15, exclude_self=True)
g = torch.Generator(device="cpu").manual_seed(0)
rows = torch.randperm(c["n"], generator=g)[:4000].cuda()
Xs = X[rows].double()
d2 = torch.cdist(Xs, X.double()) ** 2
d2[torch.arange(4000), rows] = float("inf")
thr = torch.gather(d2, 1, ei[rows].long()).sort(1).values          # 4000 x 15
C = (d2.unsqueeze(2) < thr.unsqueeze(1)).sum(1)                     # cumulative counts below t_m
B = torch.diff(torch.cat([torch.zeros_like(C[:, :1]), C], 1), dim=1)  # bucket counts
tot = C[:, -1].double()
print("mean columns below t_max per row:", tot.mean().item(), "of", c["n"])
print("mean bucket counts:", [round(v, 1) for v in B.double().mean(0).tolist()])
print("fraction of below-t_max columns in top bucket:", (B[:, -1].double().sum() / tot.sum()).item())
print("... in top 2 buckets:", (B[:, -2:].double().sum() / tot.sum()).item(), " top 3:", (B[:, -3:].double().sum() / tot.sum()).item())
q = torch.quantile(tot, torch.tensor([0.5, 0.9, 0.99], dtype=torch.float64, device=tot.device))
print("quantiles of below-t_max per row (50/90/99%):", q.tolist())
nbad = (C > 15).sum(1).double()
print("mean #thresholds with rank > k per row:", nbad.mean().item())

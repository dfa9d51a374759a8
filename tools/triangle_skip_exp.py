"""Measurement for planning (not a product path): how many 256x256 (query block, reference
tile) pairs of the trust fine pass would a triangle-inequality bound skip, versus the coarse
BF16 GEMM pass (91 of 274 tiles kept per block at C2)?  Rows and columns in a 2-D space-
filling order of the embedding; per tile: centroid c_T and radius R_T in input space; a
block skips tile T if for every row q: (|q - c_T| - R_T)^2 > t_max(q)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2008_00325_b200 as U
c = synth.CONFIGS["C2"]
X = torch.from_numpy(synth.lowrank(c["n"], c["d"], c["blobs"], c["seed"])).cuda()
Y, _ = U.fit(X, n_neighbors=15, n_epochs=500, knn_mode="tensor")
n = X.shape[0]
# Morton order of Y (16 bits per axis)
lo, hi = Y.min(0).values, Y.max(0).values
g = ((Y - lo) / (hi - lo + 1e-9) * 65535).long()
def spread(v):
    v = v & 0xFFFF
    v = (v | (v << 8)) & 0x00FF00FF
    v = (v | (v << 4)) & 0x0F0F0F0F
    v = (v | (v << 2)) & 0x33333333
    v = (v | (v << 1)) & 0x55555555
    return v
key = spread(g[:, 0]) | (spread(g[:, 1]) << 1)
perm = torch.argsort(key)
Xp = X[perm].double()
# thresholds: exact distances to the 15 embedding neighbours; t_max per row
ei, _ = U.knn(Y, Y, 15, exclude_self=True, mode="exact")
ei = ei.long()
tmax = torch.empty(n, dtype=torch.float64, device="cuda")
for s in range(0, n, 4096):
    xs = X[s:s + 4096].double()
    d2 = ((xs[:, None, :] - X[ei[s:s + 4096]].double()) ** 2).sum(-1)
    tmax[s:s + 4096] = d2.max(1).values
tmax_p = tmax[perm]
T = (n + 255) // 256
cent = torch.stack([Xp[t * 256:(t + 1) * 256].mean(0) for t in range(T)])
rad = torch.stack([((Xp[t * 256:(t + 1) * 256] - cent[t]) ** 2).sum(1).sqrt().max() for t in range(T)])
kept = 0
for b in range(T):
    q = Xp[b * 256:(b + 1) * 256]
    dqc = torch.cdist(q, cent)                     # [rows, T]
    lb = torch.clamp(dqc - rad[None, :], min=0) ** 2
    need = (lb <= tmax_p[b * 256:(b + 1) * 256, None]).any(0)
    kept += int(need.sum())
print(f"triangle bound keeps {kept / T:.1f} of {T} tiles per block (coarse GEMM pass: 91.3)")
print(f"tile radius median {rad.median().item():.1f}, centroid spacing median "
      f"{torch.cdist(cent, cent).median().item():.1f}, sqrt(t_max) median {tmax.sqrt().median().item():.1f}")

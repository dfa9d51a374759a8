"""Measurement only (no library code): would a low-dimensional projection of X prune the trust
pass's (256-row block, 256-column tile) pairs as well as the full-dimensional coarse pass?
d2_P = |P^T (x_q - x_r)|^2 <= d2 for an orthonormal P (PCA basis), so a tile whose projected
distances all exceed a row's largest threshold (plus the BF16 margin) can be skipped rigorously.
Uses an embedding dumped by tools/dump_embedding.py.   python tools/proj_prune_est.py Y_C2.npy"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from scipy.spatial import cKDTree  # noqa: E402

import synth  # noqa: E402

Y = np.load(sys.argv[1]).astype(np.float64)
c = synth.CONFIGS["C2"]
X = synth.lowrank(c["n"], c["d"], c["blobs"], c["seed"]).astype(np.float64)
n = X.shape[0]
X -= X.mean(0)
_, emb = cKDTree(Y).query(Y, 16)
emb = emb[:, 1:]
sq = (X * X).sum(1)


def hilbert_d(x, y, order=16):
    d = np.zeros_like(x)
    s = 1 << (order - 1)
    while s > 0:
        rx = ((x & s) > 0).astype(np.int64)
        ry = ((y & s) > 0).astype(np.int64)
        d += s * s * ((3 * rx) ^ ry)
        m = ry == 0
        swap = m & (rx == 1)
        x = np.where(swap, s - 1 - x, x); y = np.where(swap, s - 1 - y, y)
        x2 = np.where(m, y, x); y2 = np.where(m, x, y)
        x, y = x2, y2
        s >>= 1
    return d


g = ((Y - Y.min(0)) / (Y.max(0) - Y.min(0) + 1e-12) * 65535).astype(np.int64)
perm = np.argsort(hilbert_d(g[:, 0], g[:, 1]), kind="stable")
Xo, sqo = X[perm], sq[perm]
tmax = np.array([max(((X[i] - X[j]) ** 2).sum() for j in emb[i]) for i in range(n)])[perm]
nb = (n + 255) // 256
rng = np.random.default_rng(0)
blocks = rng.choice(nb, 12, replace=False)
samp = Xo[rng.choice(n, 8192, replace=False)]
res = {}
for K in (0, 16, 32, 64, 128):
    if K:
        _, _, Vt = np.linalg.svd(samp, full_matrices=False)
        P = Vt[:K].T
        Z = Xo @ P
        zn = (Z * Z).sum(1)
        cm = 4.5e-3  # BF16 coarse margin class
    kept = 0
    for b in blocks:
        r0, r1 = b * 256, min(n, b * 256 + 256)
        if K:
            d2 = zn[r0:r1, None] + zn[None, :] - 2 * Z[r0:r1] @ Z.T
            e = cm * (zn[r0:r1, None] + zn[None, :])
        else:
            d2 = sqo[r0:r1, None] + sqo[None, :] - 2 * Xo[r0:r1] @ Xo.T
            e = 4.5e-3 * (sqo[r0:r1, None] + sqo[None, :])
        ok = (d2 - e) <= tmax[r0:r1, None]
        tiles = np.add.reduceat(ok.any(0).astype(np.int64), np.arange(0, n, 256)) > 0
        kept += tiles.sum()
        if K == 0:  # finer granularity of the same (exact) test: 128-row halves, 128-column tiles
            for h in (0, 128):
                okh = ok[h:h + 128]
                kept_h128 = (np.add.reduceat(okh.any(0).astype(np.int64), np.arange(0, n, 256)) > 0).sum()
                kept_h64c = (np.add.reduceat(okh.any(0).astype(np.int64), np.arange(0, n, 128)) > 0).sum()
                res.setdefault("h128", 0); res.setdefault("h128c128", 0)
                res["h128"] += kept_h128; res["h128c128"] += kept_h64c
            res.setdefault("pairs", 0); res["pairs"] += ok.mean()
    res[K] = kept / (len(blocks) * nb)
    print(f"K={K or 'full'}: kept tile fraction {res[K]:.3f}", flush=True)
    if K == 0:
        print(f"  128-row halves x 256-col tiles: {res['h128'] / (2 * len(blocks) * nb):.3f};"
              f"  128-row halves x 128-col tiles: {res['h128c128'] / (2 * len(blocks) * ((n + 127) // 128)):.3f};"
              f"  pairs below threshold: {res['pairs'] / len(blocks):.4f}", flush=True)

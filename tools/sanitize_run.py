"""Tiny invocation of every kernel family of the library, for compute-sanitizer
(tools/sanitize.sh): exact and tensor kNN (+ re-rank, top-k merge), rho/sigma + membership,
fuzzy union, random and spectral init, the deterministic SGD kernels (flat3, flat2, the
round-1 flat kernel via UMAP_SGD_VARIANT), the Hogwild persistent kernel, the transform in
both precisions, trustworthiness in both modes (coarse / fine tensor passes, rank_fix,
thresholds, grid kNN), the supervised adjustment.  Synthetic seeded inputs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2008_00325_b200 as U  # noqa: E402

A_, B_ = 1.5769434603, 0.8950608779
n, d = int(os.environ.get("SAN_N", "600")), 40
X = torch.from_numpy(synth.lowrank(n, d, blobs=4, seed=1)).cuda()
Xq = torch.from_numpy(synth.lowrank(200, d, blobs=4, seed=2)).cuda()
lab = torch.from_numpy(synth.lowrank(n, 1, blobs=3, seed=3, return_labels=True)[1].astype("int32")).cuda()
ep = int(os.environ.get("SAN_EPOCHS", "12"))
for mode in ("exact", "tensor"):
    i, dd = U.knn(X, X, 15, exclude_self=True, mode=mode)
    ii, d2 = U.knn(X, X[:300], 15, exclude_self=True, index_offset=0, mode=mode, squared=True)
    ij, d3 = U.knn(X, X[300:], 15, exclude_self=True, index_offset=300, mode=mode, squared=True)
    U.topk_merge(torch.stack([ii, ij]), torch.stack([d2, d3]), 15, squared=True)
    for sgd in ("deterministic", "hogwild"):
        Y, st = U.fit(X, n_neighbors=15, n_epochs=ep, a=A_, b=B_, sgd_mode=sgd, knn_mode=mode, trust_k=10)
    for prec in ("fp32", "fp64"):
        Yq = U.transform(X, Y, Xq, n_neighbors=15, n_epochs=ep, a=A_, b=B_, knn_mode=mode, transform_precision=prec)
    print(mode, "trust", U.trustworthiness(X, Y, 10, knn_mode=mode), flush=True)
Y, st = U.fit(X, n_neighbors=15, n_epochs=ep, a=A_, b=B_, init="spectral", spectral_iters=20)
Y, st = U.fit(X, labels=lab, n_neighbors=15, n_epochs=ep, a=A_, b=B_)
for dim in (3, 16):
    Y, st = U.fit(X, n_neighbors=15, n_components=dim, n_epochs=ep, a=A_, b=B_)
print("ok", flush=True)

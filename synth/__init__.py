"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the UMAP method: it only draws input matrices.
It is the one module both the oracle side and the CUDA side may use (task rule ③).

Recipes (DESIGN.md §"Input recipe"):

* ``lowrank`` -- class-structured low-rank Gaussian mixture, intrinsic rank r=10,
  standing in for the image / expression datasets of the paper's Table 3
  (PAPER.md:210-226).  Drawn with ``numpy.random.Generator(PCG64(seed))`` in this order::

      lab = integers(0, B, n)
      C   = standard_normal((B, d)) * 3
      A   = standard_normal((B, r, d)) / sqrt(r)
      Z   = standard_normal((n, r)) * 2
      E   = standard_normal((n, d)) * 0.3
      X   = (C[lab] + einsum('nr,nrd->nd', Z, A[lab]) + E).astype(float32)

* ``iso`` -- the paper's "isotropic blobs" of Table 4:
  ``C ~ U(-10, 10)^d`` per blob, ``X = C[lab] + N(0, I)``.  Near-ties and hub
  vertices make it the stress variant.

* ``ties`` -- small integer-lattice data with exact duplicate distances, for the
  tie-by-index rule of the kNN definition.

Configs (BASELINE.json ``configs``):
C1 digits 1797x64 B=10 seed 0; C2 MNIST 70000x784 B=10 seed 1;
C3 60000x3072 B=20 seed 2; C4 1000000x50 B=30 seed 3; C5 100000x784 train +
8,000,000x784 transform, B=10 seed 4.
"""
from __future__ import annotations

import numpy as np

CONFIGS = {
    "C1": dict(n=1797, d=64, blobs=10, seed=0, k=15, n_epochs=200),
    "C2": dict(n=70000, d=784, blobs=10, seed=1, k=15, n_epochs=500),
    "C3": dict(n=60000, d=3072, blobs=20, seed=2, k=15, n_epochs=200, trust_k=5),
    "C4": dict(n=1000000, d=50, blobs=30, seed=3, k=15, n_epochs=200),
    "C5": dict(n=100000, d=784, blobs=10, seed=4, k=15, n_epochs=200, n_transform=8000000),
}


def lowrank(n: int, d: int, blobs: int = 10, seed: int = 0, rank: int = 10,
            return_labels: bool = False, row_offset: int = 0):
    """Low-rank Gaussian mixture (see module docstring). ``row_offset`` is unused by the
    recipe itself; rows are always drawn from row 0 so any prefix is reproducible."""
    del row_offset
    g = np.random.Generator(np.random.PCG64(seed))
    lab = g.integers(0, blobs, n)
    C = g.standard_normal((blobs, d)) * 3.0
    A = g.standard_normal((blobs, rank, d)) / np.sqrt(rank)
    Z = g.standard_normal((n, rank)) * 2.0
    E = g.standard_normal((n, d)) * 0.3
    X = C[lab] + E
    # per-blob low-rank part, blob by blob to bound memory
    for c in range(blobs):
        sel = np.nonzero(lab == c)[0]
        if sel.size:
            X[sel] += Z[sel] @ A[c]
    X = np.ascontiguousarray(X.astype(np.float32))
    return (X, lab) if return_labels else X


def lowrank_model(d: int, blobs: int, seed: int, rank: int = 10):
    """Blob centres C (B x d) and low-rank bases A (B x rank x d) of the lowrank recipe, from
    their own PCG64 stream, so that several samples (train rows, transform chunks) share one
    mixture: ``C = N(0,1)*3``, ``A = N(0,1)/sqrt(rank)``."""
    g = np.random.Generator(np.random.PCG64(seed))
    C = g.standard_normal((blobs, d)) * 3.0
    A = g.standard_normal((blobs, rank, d)) / np.sqrt(rank)
    return C, A


def lowrank_sample(model, n: int, seed: int, return_labels: bool = False):
    """n rows from a ``lowrank_model``: ``lab = integers(0,B,n)``, ``Z = N(0,1)^{n x r}*2``,
    ``E = N(0,1)^{n x d}*0.3``, ``X = C[lab] + Z A[lab] + E`` (fp32), drawn in that order."""
    C, A = model
    blobs, rank, d = A.shape
    g = np.random.Generator(np.random.PCG64(seed))
    lab = g.integers(0, blobs, n)
    Z = g.standard_normal((n, rank)) * 2.0
    E = g.standard_normal((n, d)).astype(np.float32) * np.float32(0.3)
    X = C[lab].astype(np.float32) + E
    for c in range(blobs):
        sel = np.nonzero(lab == c)[0]
        if sel.size:
            X[sel] += (Z[sel] @ A[c]).astype(np.float32)
    X = np.ascontiguousarray(X, dtype=np.float32)
    return (X, lab) if return_labels else X


def c5_train(n: int = 100000, d: int = 784, seed: int = 4):
    """C5 training rows: the model of seed 4, sample seed 40."""
    return lowrank_sample(lowrank_model(d, 10, seed), n, seed * 10)


def c5_transform_chunk(chunk: int, rows: int = 1000000, d: int = 784, seed: int = 4):
    """C5 transform rows, chunk by chunk (8 chunks of 1,000,000 = 8,000,000 rows): the same
    mixture as ``c5_train``, sample seed 41 + chunk."""
    return lowrank_sample(lowrank_model(d, 10, seed), rows, seed * 10 + 1 + chunk)


def lowrank_sample_device(model, n: int, seed: int, device="cuda"):
    """``lowrank_sample`` drawn on the GPU (torch Philox stream of ``seed``) for the 25 GB C5
    transform set: the same mixture and recipe, a different random stream.  Rows used for
    oracle checks are copied back, so both sides read the same bytes."""
    import torch
    C, A = model
    blobs, rank, d = A.shape
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    lab = torch.randint(0, blobs, (n,), generator=g, device=device)
    Z = torch.randn((n, rank), generator=g, device=device) * 2.0
    X = torch.randn((n, d), generator=g, device=device) * 0.3
    Ct = torch.as_tensor(C, dtype=torch.float32, device=device)
    At = torch.as_tensor(A, dtype=torch.float32, device=device)
    X += Ct[lab]
    for c in range(blobs):
        sel = torch.nonzero(lab == c).squeeze(1)
        if sel.numel():
            X[sel] += Z[sel] @ At[c]
    return X.contiguous()


def iso(n: int, d: int, blobs: int = 10, seed: int = 0, return_labels: bool = False):
    """Isotropic blobs (Table 4): centres U(-10,10)^d, unit noise."""
    g = np.random.Generator(np.random.PCG64(seed))
    lab = g.integers(0, blobs, n)
    C = g.uniform(-10.0, 10.0, (blobs, d))
    X = (C[lab] + g.standard_normal((n, d))).astype(np.float32)
    X = np.ascontiguousarray(X)
    return (X, lab) if return_labels else X


def ties(n: int, d: int, seed: int = 0, levels: int = 3):
    """Integer lattice points in {0..levels-1}^d: many exactly equal distances and
    duplicate rows, to exercise the (distance, index) tie rule."""
    g = np.random.Generator(np.random.PCG64(seed))
    return np.ascontiguousarray(g.integers(0, levels, (n, d)).astype(np.float32))


def uniform_embedding(n: int, dim: int = 2, seed: int = 0, scale: float = 10.0):
    """A random low-dimensional layout (teacher-forcing input for SGD parity tests)."""
    g = np.random.Generator(np.random.PCG64(seed))
    return np.ascontiguousarray(g.uniform(-scale, scale, (n, dim)).astype(np.float32))


def make(config: str, **overrides):
    """Input matrix for a named config (C1..C5) with the lowrank recipe."""
    c = dict(CONFIGS[config])
    c.update(overrides)
    return lowrank(c["n"], c["d"], c["blobs"], c["seed"])

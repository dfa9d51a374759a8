"""CPU oracle of the GPU-UMAP hot path (arXiv 2008.00325) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module.  The product path
(``paper_2008_00325_b200``) never imports it and shares no code with it.

Wraps ``oracle/liboracle.so`` (plain C, see ``umap_oracle.c``) with numpy, plus
the a/b curve fit (R8) done with scipy's Levenberg-Marquardt ``curve_fit`` on the
fixed 300-point grid.  Every function cites the passage it follows; the readings
R1..R18 are listed in DESIGN.md.

Parity unpinned (no value in the paper to pin them to; they are fixed only by the readings
and checked through invariants): the self-exclusion convention of knn (R1), the bracket and
tolerance of smooth_knn's bisection (R5), the closed-form schedule of optimize (R9), the
Philox stream of random_init / negative samples (R11), the s = 0 repulsion kick (R12), the
transform epoch budget (R15), spectral_init's iteration count (R18), and Hogwild
trajectories (optimize mode="hogwild", compared only through trustworthiness).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "umap_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
# tools/oracle_mutants.py points this at deliberately broken builds to show the pins catch them
_LIB_OVERRIDE = os.environ.get("UMAP_ORACLE_LIB")

_c_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_c_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_c_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_c_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_I64, _I32, _F32, _F64, _U64 = ctypes.c_int64, ctypes.c_int32, ctypes.c_float, ctypes.c_double, ctypes.c_uint64


def build(force: bool = False) -> str:
    """Compile the C oracle (gcc -O2 -ffp-contract=off -fopenmp, no fast-math)."""
    if _LIB_OVERRIDE:
        return _LIB_OVERRIDE
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        L.oracle_set_threads.restype = None
        L.oracle_get_threads.restype = ctypes.c_int
        L.oracle_philox4x32_10.argtypes = [_c_u32p, _c_u32p, _c_u32p]
        L.oracle_philox4x32_10.restype = None
        L.oracle_sqdist.argtypes = [_c_f32p, _c_f32p, _I32]
        L.oracle_sqdist.restype = ctypes.c_float
        L.oracle_knn.argtypes = [_c_f32p, _I64, _c_f32p, _I64, _I32, _I32, _I64, _c_i32p, _c_f32p]
        L.oracle_knn.restype = ctypes.c_int
        L.oracle_smooth_knn.argtypes = [_c_f32p, _I64, _I32, _c_f32p, _c_f32p]
        L.oracle_membership.argtypes = [_c_f32p, _c_f32p, _c_f32p, _I64, _I32, _c_f32p]
        L.oracle_fuzzy_union.argtypes = [_c_i32p, _c_f32p, _I64, _I32, _c_i64p, _c_i32p, _c_f32p]
        L.oracle_fuzzy_union.restype = _I64
        L.oracle_random_init.argtypes = [_I64, _I32, _U64, _c_f32p]
        L.oracle_edge_due.argtypes = [_F32, _I32]
        L.oracle_edge_due.restype = ctypes.c_int
        L.oracle_attr_coef.argtypes = [_F64, _F64, _F64]
        L.oracle_attr_coef.restype = _F64
        L.oracle_rep_coef.argtypes = [_F64, _F64, _F64, _F64]
        L.oracle_rep_coef.restype = _F64
        L.oracle_optimize.argtypes = [_c_i64p, _c_i32p, _c_f32p, _I64, _I32, _c_f32p, _F32, _F32, _F32, _F32,
                                      _I32, _I32, _I32, _I32, _U64, _I32]
        L.oracle_transform_init.argtypes = [_c_i32p, _c_f32p, _I64, _I32, _c_f32p, _I32, _c_f32p]
        L.oracle_transform_optimize.argtypes = [_c_i32p, _c_f32p, _I64, _I32, _c_f32p, _I64, _I32, _c_f32p,
                                                _F32, _F32, _F32, _F32, _I32, _I32, _U64, _I64]
        L.oracle_transform_optimize_range.argtypes = [_c_i32p, _c_f32p, _I64, _I32, _c_f32p, _I64, _I32, _c_f32p,
                                                      _F32, _F32, _F32, _F32, _I32, _I32, _I32, _I32, _U64, _I64]
        L.oracle_trust_penalty.argtypes = [_c_f32p, _I32, _c_f32p, _I32, _I64, _I32, _I64, _I64,
                                           ctypes.c_void_p]
        L.oracle_trust_penalty.restype = _I64
        L.oracle_trust_from_penalty.argtypes = [_I64, _I64, _I32]
        L.oracle_trust_from_penalty.restype = _F64
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    """OpenMP threads for the row-parallel loops (results do not depend on it)."""
    lib().oracle_set_threads(int(n))


def get_threads() -> int:
    return int(lib().oracle_get_threads())


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


# ---------------------------------------------------------------- Philox (R11)
def philox4x32_10(ctr, key):
    out = np.zeros(4, np.uint32)
    lib().oracle_philox4x32_10(np.asarray(ctr, np.uint32), np.asarray(key, np.uint32), out)
    return out


# ------------------------------------------------------------ kNN (R1, R2)
def sqdist(x, y) -> float:
    x, y = _f32(x), _f32(y)
    return float(lib().oracle_sqdist(x, y, x.shape[0]))


def knn(Xq, Xr, k: int, self_offset: int = -1):
    """Exact kNN by key (fp32 sequential-FMA d^2, index). Returns (idx int32, dist fp32)."""
    Xq, Xr = _f32(Xq), _f32(Xr)
    nq, d = Xq.shape
    idx = np.empty((nq, k), np.int32)
    dist = np.empty((nq, k), np.float32)
    lib().oracle_knn(Xq, nq, Xr, Xr.shape[0], d, k, self_offset, idx, dist)
    return idx, dist


# ----------------------------------------------------- rho, sigma, w (R4-R6)
def smooth_knn(dist):
    """Eq. 1: per-row rho and sigma."""
    dist = _f32(dist)
    n, k = dist.shape
    rho = np.empty(n, np.float32)
    sigma = np.empty(n, np.float32)
    lib().oracle_smooth_knn(dist, n, k, rho, sigma)
    return rho, sigma


def membership(dist, rho, sigma):
    """w_ij = exp(-max(0, d_ij - rho_i)/sigma_i)."""
    dist = _f32(dist)
    n, k = dist.shape
    w = np.empty((n, k), np.float32)
    lib().oracle_membership(dist, _f32(rho), _f32(sigma), n, k, w)
    return w


# ------------------------------------------------------------ union (R7)
def fuzzy_union(idx, w):
    """Eq. 2: B = A + A^T - A o A^T as CSR sorted by (row, col)."""
    idx = np.ascontiguousarray(idx, np.int32)
    w = _f32(w)
    n, k = idx.shape
    indptr = np.zeros(n + 1, np.int64)
    col = np.empty(2 * n * k, np.int32)
    val = np.empty(2 * n * k, np.float32)
    nnz = lib().oracle_fuzzy_union(idx, w, n, k, indptr, col, val)
    return indptr, col[:nnz].copy(), val[:nnz].copy()


# ------------------------------------------------------------ a, b (R8)
def fit_ab(min_dist: float = 0.1, spread: float = 1.0):
    """Fit Phi(d) = 1/(1 + a d^{2b}) (Eq. 3's "approximate form") to the
    min_dist curve y = 1 (x < min_dist), exp(-(x - min_dist)/spread) otherwise, on
    linspace(0, 3*spread, 300), by Levenberg-Marquardt from (1, 1)."""
    from scipy.optimize import curve_fit

    def curve(x, a, b):
        return 1.0 / (1.0 + a * x ** (2 * b))

    xv = np.linspace(0, spread * 3, 300)
    yv = np.zeros(xv.shape)
    yv[xv < min_dist] = 1.0
    yv[xv >= min_dist] = np.exp(-(xv[xv >= min_dist] - min_dist) / spread)
    params, _ = curve_fit(curve, xv, yv)
    return float(params[0]), float(params[1])


# ------------------------------------------------------------ SGD (R9-R14)
def random_init(n: int, dim: int, seed: int):
    Y = np.empty((n, dim), np.float32)
    lib().oracle_random_init(n, dim, seed, Y)
    return Y


def philox_vec(c0, c1, c2, c3, seed: int):
    """Philox4x32-10 (R11) vectorised over numpy uint32 counter arrays (same rounds as the C
    oracle; pinned against it by tests/test_oracle.py)."""
    M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
    W0, W1 = 0x9E3779B9, 0xBB67AE85
    c0, c1, c2, c3 = (np.asarray(x, np.uint64) & np.uint64(0xFFFFFFFF) for x in (c0, c1, c2, c3))
    k0, k1 = seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF
    mask = np.uint64(0xFFFFFFFF)
    for r in range(10):
        if r:
            k0, k1 = (k0 + W0) & 0xFFFFFFFF, (k1 + W1) & 0xFFFFFFFF
        p0, p1 = M0 * c0, M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & mask
        hi1, lo1 = p1 >> np.uint64(32), p1 & mask
        c0, c1, c2, c3 = hi1 ^ c1 ^ np.uint64(k0), lo1, hi0 ^ c3 ^ np.uint64(k1), lo0
    return c0.astype(np.uint32), c1.astype(np.uint32), c2.astype(np.uint32), c3.astype(np.uint32)


def _uniform_pm1(n, dim, seed, tag):
    """U[-1, 1) per (row, column) from Philox counter (row, column, tag, 0), first word."""
    i = np.repeat(np.arange(n, dtype=np.uint64), dim)
    c = np.tile(np.arange(dim, dtype=np.uint64), n)
    u = philox_vec(i, c, np.full(i.shape, tag, np.uint64), np.zeros(i.shape, np.uint64), seed)[0]
    return (-1.0 + 2.0 * (u >> np.uint32(8)).astype(np.float64) * 2.0 ** -24).reshape(n, dim)


def spectral_init(indptr, col, w, dim, seed=0, iters=300, scale=10.0):
    """Spectral initialisation ("computing a spectral embedding over the fuzzy union",
    P:134; reading R18): the dim eigenvectors of L = I - D^-1/2 B D^-1/2 with the
    smallest non-trivial eigenvalues, by orthogonal (block power) iteration on
    M = 2I - L = I + D^-1/2 B D^-1/2 with the trivial vector D^1/2 1 deflated, in fp64:
    V0 = U[-1,1) from Philox (row, column, 0xFFFFFFFE); `iters` times W = M V, W -= v0 (v0' W),
    V = W R^-1 with R'R = W'W (Cholesky QR).  Each column is then rescaled affinely to
    [-scale, scale] and noise 1e-4 scale U[-1,1) (counter tag 0xFFFFFFFD) is added; fp32 out."""
    indptr, col = np.asarray(indptr, np.int64), np.asarray(col, np.int64)
    w = np.asarray(w, np.float32).astype(np.float64)
    n = indptr.shape[0] - 1
    rows = np.repeat(np.arange(n), np.diff(indptr))
    deg = np.zeros(n)
    for i in range(n):  # row sums in CSR order (sequential, as the definition reads)
        s_ = 0.0
        for e in range(indptr[i], indptr[i + 1]):
            s_ += w[e]
        deg[i] = s_
    sq = np.sqrt(deg)
    dinv = np.where(sq > 0, 1.0 / np.where(sq > 0, sq, 1.0), 0.0)
    v0 = sq / np.linalg.norm(sq)
    V = _uniform_pm1(n, dim, seed, 0xFFFFFFFE)
    for _ in range(iters):
        Z = dinv[:, None] * V
        BZ = np.zeros_like(V)
        np.add.at(BZ, rows, w[:, None] * Z[col])
        W_ = V + dinv[:, None] * BZ
        d0 = v0 @ W_
        W_ = W_ - np.outer(v0, d0)
        G = W_.T @ W_
        R = np.linalg.cholesky(G).T
        V = W_ @ np.linalg.inv(R)
    lo, hi = V.min(0), V.max(0)
    span = np.where(hi > lo, hi - lo, 1.0)
    Y = (V - lo) / span * (2.0 * scale) - scale
    Y = Y + 1e-4 * scale * _uniform_pm1(n, dim, seed, 0xFFFFFFFD)
    return Y.astype(np.float32), V


def edge_due(r: float, e: int) -> bool:
    return bool(lib().oracle_edge_due(np.float32(r), e))


def attr_coef(s, a, b):
    return lib().oracle_attr_coef(s, a, b)


def rep_coef(s, a, b, gamma=1.0):
    return lib().oracle_rep_coef(s, a, b, gamma)


def optimize(indptr, col, w, Y, a, b, n_epochs, e_begin=1, e_end=None, m=5, seed=0,
             mode="deterministic", gamma=1.0, alpha0=1.0):
    """SGD layout over the union. Returns a new Y (input not modified)."""
    Y = np.array(Y, dtype=np.float32, order="C", copy=True)
    n, dim = Y.shape
    if e_end is None:
        e_end = n_epochs
    lib().oracle_optimize(np.ascontiguousarray(indptr, np.int64), np.ascontiguousarray(col, np.int32),
                          _f32(w), n, dim, Y, a, b, gamma, alpha0, n_epochs, e_begin, e_end, m, seed,
                          1 if mode == "deterministic" else 0)
    return Y


def transform_init(idx, w, Ytr):
    idx = np.ascontiguousarray(idx, np.int32)
    nq, k = idx.shape
    Ytr = _f32(Ytr)
    Yq = np.empty((nq, Ytr.shape[1]), np.float32)
    lib().oracle_transform_init(idx, _f32(w), nq, k, Ytr, Ytr.shape[1], Yq)
    return Yq


def transform_optimize(idx, w, Ytr, Yq, a, b, n_epochs_t, m=5, seed=0, q_offset=0, gamma=1.0, alpha0=1.0,
                       e_begin=1, e_end=None):
    """Query-row SGD, epochs [e_begin, e_end) of an N_t = n_epochs_t schedule."""
    idx = np.ascontiguousarray(idx, np.int32)
    nq, k = idx.shape
    Ytr = _f32(Ytr)
    Yq = np.array(Yq, dtype=np.float32, order="C", copy=True)
    if e_end is None:
        e_end = n_epochs_t
    lib().oracle_transform_optimize_range(idx, _f32(w), nq, k, Ytr, Ytr.shape[0], Ytr.shape[1], Yq, a, b, gamma,
                                          alpha0, n_epochs_t, e_begin, e_end, m, seed, q_offset)
    return Yq


# ------------------------------------------------------------ trust (R16)
def trust_penalty(X, Y, k, row_begin=0, row_end=None):
    X, Y = _f32(X), _f32(Y)
    n = X.shape[0]
    if row_end is None:
        row_end = n
    pen = np.zeros(row_end - row_begin, np.int64)
    S = lib().oracle_trust_penalty(X, X.shape[1], Y, Y.shape[1], n, k, row_begin, row_end,
                                   pen.ctypes.data_as(ctypes.c_void_p))
    return int(S), pen


def trust_from_penalty(S, n, k):
    return float(lib().oracle_trust_from_penalty(S, n, k))


def trustworthiness(X, Y, k):
    S, _ = trust_penalty(X, Y, k)
    return trust_from_penalty(S, X.shape[0], k)


# ------------------------------------------------------------ pipelines
DEFAULTS = dict(k=15, n_components=2, min_dist=0.1, spread=1.0, m=5, gamma=1.0, alpha0=1.0)


def default_epochs(n):
    """500 epochs when n <= 10000 else 200."""
    return 500 if n <= 10000 else 200


def fuzzy_graph(X, k):
    idx, dist = knn(X, X, k, self_offset=0)
    rho, sigma = smooth_knn(dist)
    w = membership(dist, rho, sigma)
    return idx, dist, rho, sigma, w, fuzzy_union(idx, w)


def supervised_adjust(indptr, col, w, labels, far_dist=5.0, unknown_dist=1.0):
    """Label adjustment of the fuzzy union ("adjusts the membership strengths of the
    fuzzy sets based on their labels"; rule of SPEC S:308-316, reading R17): entry (i, j) is
    multiplied by 1 if labels[i] == labels[j] (both known), by exp(-far_dist) if both are
    known and differ, by exp(-unknown_dist) if either is -1; entries below 1e-8 are dropped.
    The factors are rounded to fp32 once, the products are fp32."""
    indptr, col, w = np.asarray(indptr, np.int64), np.asarray(col, np.int32), np.asarray(w, np.float32)
    labels = np.asarray(labels, np.int64)
    f_far, f_unk = np.float32(math.exp(-far_dist)), np.float32(math.exp(-unknown_dist))
    n = indptr.shape[0] - 1
    rows = np.repeat(np.arange(n), np.diff(indptr))
    li, lj = labels[rows], labels[col]
    factor = np.where((li < 0) | (lj < 0), f_unk, np.where(li == lj, np.float32(1.0), f_far)).astype(np.float32)
    w2 = (w * factor).astype(np.float32)
    keep = w2 >= np.float32(1e-8)
    new_indptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rows[keep], minlength=n), out=new_indptr[1:])
    return new_indptr, col[keep].copy(), w2[keep].copy()


def fit(X, k=15, n_components=2, n_epochs=None, a=None, b=None, min_dist=0.1, spread=1.0, m=5, seed=0,
        mode="deterministic", labels=None, far_dist=5.0, unknown_dist=1.0, init="random", spectral_iters=300):
    """Whole fit: kNN -> rho/sigma -> membership -> union -> (labels: supervised adjustment)
    -> init -> SGD."""
    X = _f32(X)
    n = X.shape[0]
    if n_epochs is None:
        n_epochs = default_epochs(n)
    if a is None or b is None:
        a, b = fit_ab(min_dist, spread)
    _, _, _, _, _, (indptr, col, w) = fuzzy_graph(X, k)
    if labels is not None:
        indptr, col, w = supervised_adjust(indptr, col, w, labels, far_dist, unknown_dist)
    if init == "spectral":
        Y0, _ = spectral_init(indptr, col, w, n_components, seed, spectral_iters)
    else:
        Y0 = random_init(n, n_components, seed)
    return optimize(indptr, col, w, Y0, np.float32(a), np.float32(b), n_epochs, m=m, seed=seed, mode=mode)


def transform(X_train, Y_train, Xq, k=15, n_epochs=200, a=None, b=None, m=5, seed=0, q_offset=0):
    """Out-of-sample embedding against the frozen training layout."""
    if a is None or b is None:
        a, b = fit_ab()
    idx, dist = knn(Xq, X_train, k, self_offset=-1)
    rho, sigma = smooth_knn(dist)
    w = membership(dist, rho, sigma)
    Yq = transform_init(idx, w, Y_train)
    n_t = int(math.ceil(n_epochs / 3.0))
    return transform_optimize(idx, w, Y_train, Yq, np.float32(a), np.float32(b), n_t, m=m, seed=seed,
                              q_offset=q_offset)

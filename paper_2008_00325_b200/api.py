"""Thin torch binding of the C ABI: checks dtypes/devices/contiguity, allocates
outputs with torch, passes raw pointers and the current CUDA stream.  Every step
of the hot path runs in libumapb200.so; nothing here computes.
"""
from __future__ import annotations

import contextlib
import ctypes

import torch

from . import _lib
from ._lib import UmapFitStats, UmapParams, check

SGD_MODES = {"hogwild": _lib.SGD_HOGWILD, "deterministic": _lib.SGD_DETERMINISTIC}
KNN_MODES = {"exact": _lib.KNN_EXACT_FP32, "tensor": _lib.KNN_TENSOR_BF16}


def _stream(device=None):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _call(device, name, *args):
    """Call C entry point `name`(*args, stream) with `device` current and its current stream."""
    with _on(device):
        check(getattr(_lib.load(), name)(*args, _stream(device)), name)


def _on(device):
    """Make `device` current for the C call (the library launches on the current device)."""
    if device is None or (isinstance(device, torch.device) and device.type != "cuda"):
        return contextlib.nullcontext()
    return torch.cuda.device(device)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _dev(t, dtype, name):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    return t.contiguous()


def _any(t, dtype, name):
    """CUDA tensor or (preferably pinned) CPU tensor: the C ABI stages host arrays itself."""
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    return t.contiguous()


def params(n_neighbors=15, n_components=2, n_epochs=0, min_dist=0.1, spread=1.0, negative_sample_rate=5,
           learning_rate=1.0, repulsion_strength=1.0, a=0.0, b=0.0, seed=0, sgd_mode="deterministic",
           knn_mode="exact", knn_candidates=32, transform_epochs=0, trust_k=0, far_dist=5.0,
           unknown_dist=1.0, init="random", spectral_iters=0, transform_precision="fp32") -> UmapParams:
    p = UmapParams()
    _lib.load().umap_params_default(ctypes.byref(p))
    p.n_neighbors, p.n_components, p.n_epochs = n_neighbors, n_components, n_epochs
    p.min_dist, p.spread, p.negative_sample_rate = min_dist, spread, negative_sample_rate
    p.learning_rate, p.repulsion_strength, p.a, p.b = learning_rate, repulsion_strength, a, b
    p.seed = seed
    p.sgd_mode = SGD_MODES[sgd_mode] if isinstance(sgd_mode, str) else sgd_mode
    p.knn_mode = KNN_MODES[knn_mode] if isinstance(knn_mode, str) else knn_mode
    p.knn_candidates, p.transform_epochs, p.trust_k = knn_candidates, transform_epochs, trust_k
    p.far_dist, p.unknown_dist = far_dist, unknown_dist
    p.init = {"random": 0, "spectral": 1}[init] if isinstance(init, str) else init
    p.spectral_iters = spectral_iters
    p.transform_precision = {"fp32": 0, "fp64": 1}[transform_precision] if isinstance(transform_precision, str) \
        else transform_precision
    return p


def fit_ab(min_dist=0.1, spread=1.0):
    a, b = ctypes.c_float(), ctypes.c_float()
    check(_lib.load().umap_fit_ab(min_dist, spread, ctypes.byref(a), ctypes.byref(b)), "umap_fit_ab")
    return a.value, b.value


def fit(X, out=None, labels=None, **kw):
    """umap_fit: X (n x d fp32, CUDA or CPU tensor) -> (Y, stats dict). Y lives where X lives
    unless `out` is given.  trust_k > 0 also scores Y (stats["trustworthiness"]).  labels (n
    int32, -1 = unknown): the supervised fit umap_fit_supervised (far_dist, unknown_dist)."""
    X = _any(X, torch.float32, "X")
    if labels is not None:
        labels = _any(labels, torch.int32, "labels")
    p = params(**kw)
    n, d = X.shape
    if out is None:
        out = torch.empty((n, p.n_components), dtype=torch.float32, device=X.device,
                          pin_memory=(not X.is_cuda and X.is_pinned()))
    st = UmapFitStats()
    dev = X.device if X.is_cuda else out.device if out.is_cuda else None
    if labels is None:
        _call(dev, "umap_fit", _ptr(X), n, d, ctypes.byref(p), _ptr(out), ctypes.byref(st))
    else:
        _call(dev, "umap_fit_supervised", _ptr(X), n, d, _ptr(labels), ctypes.byref(p), _ptr(out),
                                              ctypes.byref(st))
    return out, st.as_dict()


def spectral_init(indptr, col, val, dim=2, seed=0, iters=300):
    """umap_spectral_init on a device CSR graph -> Y (n x dim fp32, device)."""
    indptr = _dev(indptr, torch.int64, "indptr")
    col = _dev(col, torch.int32, "col")
    val = _dev(val, torch.float32, "val")
    n = indptr.shape[0] - 1
    Y = torch.empty((n, dim), dtype=torch.float32, device=indptr.device)
    _call(indptr.device, "umap_spectral_init", _ptr(indptr), _ptr(col), _ptr(val), n, dim, seed, iters, _ptr(Y))
    return Y


def supervised_adjust(indptr, col, val, labels, far_dist=5.0, unknown_dist=1.0):
    """umap_supervised_adjust on a device CSR -> (indptr, col, val) of the label-adjusted graph."""
    indptr = _dev(indptr, torch.int64, "indptr")
    col = _dev(col, torch.int32, "col")
    val = _dev(val, torch.float32, "val")
    labels = _dev(labels, torch.int32, "labels")
    n = indptr.shape[0] - 1
    cap = col.shape[0]
    oi = torch.empty_like(indptr)
    oc = torch.empty_like(col)
    ov = torch.empty_like(val)
    nnz = ctypes.c_int64()
    _call(indptr.device, "umap_supervised_adjust", _ptr(indptr), _ptr(col), _ptr(val), n, _ptr(labels), far_dist,
                                             unknown_dist, _ptr(oi), _ptr(oc), _ptr(ov), cap, ctypes.byref(nnz))
    return oi, oc[:nnz.value], ov[:nnz.value]


def fit_knn(knn_idx, knn_dist, out=None, **kw):
    """umap_fit_knn: fit from a pre-computed kNN graph (App. A.1) -> (Y, stats)."""
    knn_idx = _any(knn_idx, torch.int32, "knn_idx")
    knn_dist = _any(knn_dist, torch.float32, "knn_dist")
    n, k = knn_idx.shape
    p = params(n_neighbors=k, **kw)
    if out is None:
        out = torch.empty((n, p.n_components), dtype=torch.float32, device=knn_idx.device)
    st = UmapFitStats()
    dev = next((t.device for t in (knn_idx, out) if t.is_cuda), None)
    _call(dev, "umap_fit_knn", _ptr(knn_idx), _ptr(knn_dist), n, ctypes.byref(p), _ptr(out), ctypes.byref(st))
    return out, st.as_dict()


def transform(X_train, Y_train, Xq, q_offset=0, out=None, **kw):
    X_train = _any(X_train, torch.float32, "X_train")
    Y_train = _any(Y_train, torch.float32, "Y_train")
    Xq = _any(Xq, torch.float32, "Xq")
    p = params(n_components=Y_train.shape[1], **kw)
    if out is None:
        out = torch.empty((Xq.shape[0], p.n_components), dtype=torch.float32, device=Xq.device)
    dev = next((t.device for t in (Xq, X_train, out) if t.is_cuda), None)
    _call(dev, "umap_transform", _ptr(X_train), _ptr(Y_train), X_train.shape[0], X_train.shape[1], _ptr(Xq),
                                     Xq.shape[0], q_offset, ctypes.byref(p), _ptr(out))
    return out


def trustworthiness(X, Y, k=15, knn_mode="exact"):
    X = _any(X, torch.float32, "X")
    Y = _any(Y, torch.float32, "Y")
    T, S = ctypes.c_double(), ctypes.c_int64()
    dev = next((t.device for t in (X, Y) if t.is_cuda), None)
    _call(dev, "umap_trustworthiness", _ptr(X), X.shape[1], _ptr(Y), Y.shape[1], X.shape[0], k,
                                           KNN_MODES[knn_mode], ctypes.byref(T), ctypes.byref(S))
    return T.value, S.value


# ------------------------------------------------------------ building blocks
def knn(Xq, Xr, k, exclude_self=False, query_offset=0, index_offset=0, mode="exact", squared=False):
    """kNN of Xq against Xr. Global ids: query i = query_offset + i, reference j = index_offset + j;
    exclude_self drops the reference with the query's own global id. Returns (idx int32, dist fp32)."""
    Xq = _dev(Xq, torch.float32, "Xq")
    Xr = _dev(Xr, torch.float32, "Xr")
    nq, d = Xq.shape
    idx = torch.empty((nq, k), dtype=torch.int32, device=Xq.device)
    dist = torch.empty((nq, k), dtype=torch.float32, device=Xq.device)
    _call(Xq.device, "umap_knn", _ptr(Xq), nq, _ptr(Xr), Xr.shape[0], d, k, query_offset, index_offset,
                               int(exclude_self), KNN_MODES[mode] if isinstance(mode, str) else mode, int(squared),
                               _ptr(idx),
                               _ptr(dist))
    return idx, dist


def topk_merge(idx_parts, d2_parts, k_out, squared=False):
    """idx_parts/d2_parts: (n_parts, n, k_in) tensors of per-part sorted candidates."""
    idx_parts = _dev(idx_parts, torch.int32, "idx_parts")
    d2_parts = _dev(d2_parts, torch.float32, "d2_parts")
    n_parts, n, k_in = idx_parts.shape
    idx = torch.empty((n, k_out), dtype=torch.int32, device=idx_parts.device)
    dist = torch.empty((n, k_out), dtype=torch.float32, device=idx_parts.device)
    _call(idx_parts.device, "umap_topk_merge", _ptr(idx_parts), _ptr(d2_parts), n_parts, n, k_in, k_out, int(squared),
                                      _ptr(idx), _ptr(dist))
    return idx, dist


def smooth_knn(dist, idx=None, sort_by_col=False):
    """Returns (rho, sigma, w[, col_sorted_idx])."""
    dist = _dev(dist, torch.float32, "dist")
    n, k = dist.shape
    rho = torch.empty(n, dtype=torch.float32, device=dist.device)
    sigma = torch.empty_like(rho)
    w = torch.empty_like(dist)
    cs = None
    if sort_by_col:
        idx = _dev(idx, torch.int32, "idx")
        cs = torch.empty_like(idx)
    _call(dist.device, "umap_smooth_knn", _ptr(dist), _ptr(idx) if idx is not None else ctypes.c_void_p(0), n, k,
                                      _ptr(rho), _ptr(sigma), _ptr(w), _ptr(cs))
    return (rho, sigma, w, cs) if sort_by_col else (rho, sigma, w)


def fuzzy_union(col_sorted_idx, w):
    idx = _dev(col_sorted_idx, torch.int32, "idx")
    w = _dev(w, torch.float32, "w")
    n, k = idx.shape
    cap = 2 * n * k
    indptr = torch.empty(n + 1, dtype=torch.int64, device=idx.device)
    col = torch.empty(cap, dtype=torch.int32, device=idx.device)
    val = torch.empty(cap, dtype=torch.float32, device=idx.device)
    nnz = ctypes.c_int64()
    _call(idx.device, "umap_fuzzy_union", _ptr(idx), _ptr(w), n, k, _ptr(indptr), _ptr(col), _ptr(val), cap,
                                       ctypes.byref(nnz))
    return indptr, col[:nnz.value], val[:nnz.value]


def random_init(n, dim, seed, device="cuda"):
    Y = torch.empty((n, dim), dtype=torch.float32, device=device)
    _call(Y.device, "umap_random_init", n, dim, seed, _ptr(Y))
    return Y


def optimize(indptr, col, val, Y, e_begin=1, e_end=None, **kw):
    """In-place SGD over epochs [e_begin, e_end) of an N = n_epochs schedule. Returns #positives."""
    indptr = _dev(indptr, torch.int64, "indptr")
    col = _dev(col, torch.int32, "col")
    val = _dev(val, torch.float32, "val")
    if not (Y.is_cuda and Y.dtype == torch.float32 and Y.is_contiguous()):
        raise TypeError("Y must be a contiguous CUDA float32 tensor (updated in place)")
    p = params(n_components=Y.shape[1], **kw)
    if e_end is None:
        e_end = p.n_epochs
    pos = ctypes.c_int64()
    _call(Y.device, "umap_optimize", _ptr(indptr), _ptr(col), _ptr(val), Y.shape[0], _ptr(Y), ctypes.byref(p),
                                    e_begin, e_end, ctypes.byref(pos))
    return pos.value


def transform_optimize(idx, w, Y_train, Yq, n_epochs_t, e_begin=1, e_end=None, q_offset=0, init=False, **kw):
    idx = _dev(idx, torch.int32, "idx")
    w = _dev(w, torch.float32, "w")
    Y_train = _dev(Y_train, torch.float32, "Y_train")
    if not (Yq.is_cuda and Yq.dtype == torch.float32 and Yq.is_contiguous()):
        raise TypeError("Yq must be a contiguous CUDA float32 tensor (updated in place)")
    p = params(n_components=Y_train.shape[1], **kw)
    if e_end is None:
        e_end = n_epochs_t
    _call(Yq.device, "umap_transform_optimize", _ptr(idx), _ptr(w), idx.shape[0], idx.shape[1], _ptr(Y_train),
                                              Y_train.shape[0], _ptr(Yq), ctypes.byref(p), n_epochs_t, e_begin,
                                              e_end, q_offset, int(init))
    return Yq


def trust_penalty(X, emb_idx, k, row_begin=0, row_end=None, knn_mode="exact", Y=None):
    """umap_trust_penalty: integer rank penalty of rows [row_begin, row_end).  Y (optional,
    the n x 2 embedding) lets the tensor path visit rows in cluster order (same result)."""
    X = _dev(X, torch.float32, "X")
    emb_idx = _dev(emb_idx, torch.int32, "emb_idx")
    if Y is not None:
        Y = _dev(Y, torch.float32, "Y")
    n = X.shape[0]
    if row_end is None:
        row_end = n
    pen = torch.empty(row_end - row_begin, dtype=torch.int64, device=X.device)
    S = ctypes.c_int64()
    _call(X.device, "umap_trust_penalty", _ptr(X), n, X.shape[1], _ptr(emb_idx), k, row_begin, row_end,
                                         KNN_MODES[knn_mode], _ptr(Y), Y.shape[1] if Y is not None else 0,
                                         _ptr(pen),
                                         ctypes.byref(S))
    return S.value, pen


def trust_from_penalty(S, n, k):
    """umap_trust_from_penalty (R16 normaliser, computed in the C library)."""
    return float(_lib.load().umap_trust_from_penalty(int(S), int(n), int(k)))


def default_transform_epochs(n_epochs, transform_epochs=0, n_train=0):
    """umap_transform_epoch_count (R15 budget, computed in the C library)."""
    return int(_lib.load().umap_transform_epoch_count(int(n_epochs), int(transform_epochs), int(n_train)))


def kernel_launch_count():
    return int(_lib.load().umap_kernel_launch_count())


def trust_ambiguous_count():
    """pairs the last tensor-mode trust call re-checked exactly (diagnostic)."""
    return int(_lib.load().umap_trust_ambiguous_count())


def trust_fine_fraction():
    """fraction of tiles the split-precision trust pass visited in the last call (diagnostic)."""
    return float(_lib.load().umap_trust_fine_fraction())


def profile_begin():
    """start live per-kernel CUDA-event timing of this thread's launches"""
    _lib.load().umap_profile_begin()


def profile_end():
    """stop timing; {kernel slot name: (total ms, launches)} for every slot that ran"""
    L = _lib.load()
    n = 32
    ms = (ctypes.c_double * n)()
    cnt = (ctypes.c_int64 * n)()
    k = min(n, int(L.umap_profile_end(ms, cnt, n)))
    return {L.umap_profile_slot_name(i).decode(): (ms[i], int(cnt[i])) for i in range(k) if cnt[i]}


def version():
    return _lib.load().umap_version().decode()

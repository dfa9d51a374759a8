"""GPU-vs-oracle parity through the C ABI (task rule ③).  Run on a B200: pytest -m gpu.

Tolerances (BASELINE.json north_star):
  kNN exact mode ............ indices and distances bit-exact
  rho ........................ bit-exact;  sigma <= 1 fp32 ulp
  fuzzy weights .............. <= 1e-5 relative, CSR structure identical
  deterministic SGD .......... <= 1e-4 absolute per epoch (teacher-forced)
  Hogwild / end-to-end ....... trustworthiness within 0.005 of the oracle
  trustworthiness (exact) .... integer penalty identical
"""
import math

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # the marker deselects these on CPU runs; be explicit anyway
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2008_00325_b200 as U  # noqa: E402

A_, B_ = 1.5769434603, 0.8950608779
DEV = "cuda"


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def np_(t):
    return t.detach().cpu().numpy()


def ulp_diff(a, b):
    a = np.asarray(a, np.float32).view(np.int32).astype(np.int64)
    b = np.asarray(b, np.float32).view(np.int32).astype(np.int64)
    return np.abs(a - b)


# ------------------------------------------------------------------- kNN (a2)
KNN_CASES = [
    # (n, d, k, data)  -- several 128-row tiles, ragged row tails and ragged 16-feature K tails
    (1000, 50, 15, "lowrank"),
    (700, 784, 15, "lowrank"),
    (517, 64, 1, "lowrank"),
    (900, 33, 33, "iso"),
    (400, 8, 64, "lowrank"),
    (600, 3, 15, "ties"),
    (129, 17, 15, "ties"),
    (20, 5, 19, "lowrank"),
    (5000, 2, 15, "lowrank"),   # 2-D: exact uniform-grid path
    (3000, 2, 32, "iso"),
    (1000, 2, 15, "ties"),
    (40, 2, 7, "ties"),
]


def _data(kind, n, d, seed=0):
    if kind == "lowrank":
        return synth.lowrank(n, d, blobs=5, seed=seed)
    if kind == "iso":
        return synth.iso(n, d, blobs=5, seed=seed)
    return synth.ties(n, d, seed=seed)


@pytest.mark.parametrize("n,d,k,kind", KNN_CASES)
def test_knn_exact_bitexact(O, n, d, k, kind):
    X = _data(kind, n, d)
    ri, rd = O.knn(X, X, k, self_offset=0)
    gi, gd = U.knn(cu(X), cu(X), k, exclude_self=True)
    assert np.array_equal(np_(gi), ri)
    assert np.array_equal(np_(gd).view(np.int32), rd.view(np.int32))


def test_knn_exact_query_vs_reference_offsets(O):
    X = synth.lowrank(1500, 40, seed=1)
    Xq, Xr = X[:230], X[230:]
    ri, rd = O.knn(Xq, Xr, 12, self_offset=-1)
    gi, gd = U.knn(cu(Xq), cu(Xr), 12, index_offset=1000)
    assert np.array_equal(np_(gi), ri + 1000)
    assert np.array_equal(np_(gd), rd)
    gi2, gd2 = U.knn(cu(Xq), cu(Xr), 12, squared=True)
    assert np.array_equal(np.sqrt(np_(gd2)), rd)


def test_knn_split_reference_and_topk_merge(O):
    # few queries vs many references exercises the split-R path (merge kernel)
    X = synth.lowrank(6000, 24, seed=2)
    Xq = X[:40]
    ri, rd = O.knn(Xq, X, 15, self_offset=0)
    gi, gd = U.knn(cu(Xq), cu(X), 15, exclude_self=True)
    assert np.array_equal(np_(gi), ri) and np.array_equal(np_(gd), rd)
    # explicit shard merge: 3 reference shards with global ids, squared distances
    parts_i, parts_d = [], []
    bounds = [0, 1700, 4100, 6000]
    for s in range(3):
        lo, hi = bounds[s], bounds[s + 1]
        pi, pd = U.knn(cu(Xq), cu(X[lo:hi]), 15, exclude_self=True, query_offset=0, index_offset=lo,
                       squared=True)
        parts_i.append(pi)
        parts_d.append(pd)
    mi, md = U.topk_merge(torch.stack(parts_i), torch.stack(parts_d), 15)
    assert np.array_equal(np_(mi), ri) and np.array_equal(np_(md), rd)


# tensor-core candidate mode (R3): recall >= 0.999 against the exact oracle, and rows whose
# candidate set covers the truth are bit-identical to the exact mode
TC_CASES = [
    (1000, 50, 15, "lowrank"),
    (2000, 784, 15, "lowrank"),
    (1500, 100, 15, "iso"),
    (700, 3072, 15, "lowrank"),
    (300, 8, 5, "lowrank"),
    (1300, 64, 32, "lowrank"),
    (600, 3, 15, "ties"),
]


def _recall(gi, ri):
    return np.mean([len(set(a) & set(b)) / len(b) for a, b in zip(gi, ri)])


@pytest.mark.parametrize("n,d,k,kind", TC_CASES)
def test_knn_tensor_recall_and_exactness(O, n, d, k, kind):
    X = _data(kind, n, d, seed=11)
    ri, rd = O.knn(X, X, k, self_offset=0)
    gi, gd = U.knn(cu(X), cu(X), k, exclude_self=True, mode="tensor")
    gi, gd = np_(gi), np_(gd)
    assert _recall(gi, ri) >= 0.999
    same = np.array([set(a) == set(b) for a, b in zip(gi, ri)])
    assert np.array_equal(gi[same], ri[same])
    assert np.array_equal(gd[same], rd[same])


def test_knn_tensor_query_set_offsets_and_splits(O):
    X = synth.lowrank(5000, 96, seed=12)
    Xq, Xr = X[:37], X[37:]
    ri, rd = O.knn(Xq, Xr, 15)
    gi, gd = U.knn(cu(Xq), cu(Xr), 15, index_offset=500, mode="tensor")
    assert _recall(np_(gi) - 500, ri) >= 0.999
    # shard of a self-kNN: queries are global rows 0..36, references global rows 37..4999
    ri2, _ = O.knn(X[:37], X, 15, self_offset=0)
    gi2, _ = U.knn(cu(X[:37]), cu(X), 15, exclude_self=True, mode="tensor")
    assert _recall(np_(gi2), ri2) >= 0.999


def test_knn_empty_query_and_errors():
    X = cu(synth.lowrank(50, 4))
    gi, gd = U.knn(X[:0], X, 5)
    assert gi.shape == (0, 5)
    with pytest.raises(RuntimeError):
        U.knn(X, X, 50, exclude_self=True)  # k > n - 1


# ------------------------------------------------------------------- rho/sigma/w (a3, a4)
@pytest.mark.parametrize("n,d,k", [(1000, 30, 15), (333, 10, 5), (500, 64, 50), (260, 4, 2)])
def test_smooth_knn_parity(O, n, d, k):
    X = synth.lowrank(n, d, seed=3)
    idx, dist = O.knn(X, X, k, self_offset=0)
    rho, sigma = O.smooth_knn(dist)
    w = O.membership(dist, rho, sigma)
    g_rho, g_sigma, g_w, g_cs = U.smooth_knn(cu(dist), cu(idx), sort_by_col=True)
    assert np.array_equal(np_(g_rho), rho)
    assert ulp_diff(np_(g_sigma), sigma).max() <= 1
    # column-sorted rows: same (col, w) pairs re-ordered
    order = np.argsort(idx, axis=1, kind="stable")
    assert np.array_equal(np_(g_cs), np.take_along_axis(idx, order, 1))
    gw = np_(g_w)
    ref = np.take_along_axis(w, order, 1)
    assert np.all(np.abs(gw - ref) <= 1e-5 * np.abs(ref))
    _, _, g_w2 = U.smooth_knn(cu(dist))
    assert np.all(np.abs(np_(g_w2) - w) <= 1e-5 * np.abs(w))


def test_smooth_knn_degenerate_rows(O):
    dist = np.array([[0, 0, 0, 0], [2.5, 2.5, 2.5, 2.5], [0, 1, 2, 3], [1, 2, 2, 2]], np.float32)
    idx = np.array([[1, 2, 3, 0], [0, 2, 3, 1], [0, 1, 3, 2], [0, 1, 2, 3]], np.int32)
    rho, sigma = O.smooth_knn(dist)
    g_rho, g_sigma, g_w = U.smooth_knn(cu(dist), cu(idx))
    assert np.array_equal(np_(g_rho), rho) and ulp_diff(np_(g_sigma), sigma).max() <= 1
    assert np.allclose(np_(g_w), O.membership(dist, rho, sigma), rtol=1e-5)


# ------------------------------------------------------------------- union (a5)
@pytest.mark.parametrize("n,d,k,kind", [(1200, 20, 15, "lowrank"), (900, 64, 15, "iso"), (300, 3, 10, "ties")])
def test_fuzzy_union_parity(O, n, d, k, kind):
    X = _data(kind, n, d, seed=4)
    idx, dist = O.knn(X, X, k, self_offset=0)
    rho, sigma = O.smooth_knn(dist)
    w = O.membership(dist, rho, sigma)
    r_indptr, r_col, r_val = O.fuzzy_union(idx, w)
    order = np.argsort(idx, axis=1, kind="stable")
    cs = np.take_along_axis(idx, order, 1)
    ws = np.take_along_axis(w, order, 1)
    g_indptr, g_col, g_val = U.fuzzy_union(cu(cs), cu(ws))
    assert np.array_equal(np_(g_indptr), r_indptr)
    assert np.array_equal(np_(g_col), r_col)
    assert np.all(np.abs(np_(g_val) - r_val) <= 1e-5 * r_val)


def test_fuzzy_union_hub_rows(O):
    # a hub: row 0 at the origin, the others at radius ~1 in random directions of a
    # 50-D space (nearly orthogonal, mutual distance ~1.4): row 0 is everybody's
    # nearest neighbour, so A^T row 0 is far longer than a warp
    rng = np.random.default_rng(0)
    X = rng.standard_normal((400, 50)).astype(np.float32)
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    X *= rng.uniform(1, 1.1, (400, 1)).astype(np.float32)
    X[0] = 0
    idx, dist = O.knn(X, X, 8, self_offset=0)
    assert (idx == 0).sum() > 64
    rho, sigma = O.smooth_knn(dist)
    w = O.membership(dist, rho, sigma)
    r = O.fuzzy_union(idx, w)
    order = np.argsort(idx, axis=1, kind="stable")
    g = U.fuzzy_union(cu(np.take_along_axis(idx, order, 1)), cu(np.take_along_axis(w, order, 1)))
    assert np.array_equal(np_(g[0]), r[0]) and np.array_equal(np_(g[1]), r[1])
    assert np.all(np.abs(np_(g[2]) - r[2]) <= 1e-5 * r[2])


# ------------------------------------------------------------------- init (a7)
def test_random_init_bitexact(O):
    for dim, seed in [(2, 0), (3, 12345678901234), (16, 7)]:
        assert np.array_equal(np_(U.random_init(3001, dim, seed)), O.random_init(3001, dim, seed))


# ------------------------------------------------------------------- SGD (a6, a8)
def _graph(O, n=1500, d=32, k=15, seed=5, kind="lowrank"):
    X = _data(kind, n, d, seed=seed)
    _, _, _, _, _, (indptr, col, val) = O.fuzzy_graph(X, k)
    return X, indptr, col, val


@pytest.mark.parametrize("kind", ["lowrank", "iso"])
def test_sgd_deterministic_teacher_forced(O, kind):
    X, indptr, col, val = _graph(O, kind=kind)
    n = X.shape[0]
    N = 200
    Y = synth.uniform_embedding(n, 2, seed=1)
    for e in (1, 2, 57, 120, 199):
        ref = O.optimize(indptr, col, val, Y, A_, B_, N, e_begin=e, e_end=e + 1, m=5, seed=11)
        Yg = cu(Y)
        U.optimize(cu(indptr), cu(col), cu(val), Yg, e_begin=e, e_end=e + 1, n_epochs=N, a=A_, b=B_, seed=11,
                   sgd_mode="deterministic")
        err = np.abs(np_(Yg) - ref).max()
        assert err <= 1e-4, (e, err)
        Y = ref  # teacher forcing: next epoch starts from the oracle's state


def test_sgd_deterministic_reproducible_and_dims(O):
    X, indptr, col, val = _graph(O, n=900)
    for dim in (2, 3, 16):
        Y0 = cu(synth.uniform_embedding(900, dim, seed=2))
        outs = []
        for _ in range(2):
            Yg = Y0.clone()
            U.optimize(cu(indptr), cu(col), cu(val), Yg, e_begin=1, e_end=30, n_epochs=30, a=A_, b=B_, seed=3)
            outs.append(np_(Yg))
        assert np.array_equal(outs[0], outs[1])
        ref = O.optimize(indptr, col, val, np_(Y0), A_, B_, 30, e_begin=5, e_end=6, m=5, seed=3)
        Yg = Y0.clone()
        U.optimize(cu(indptr), cu(col), cu(val), Yg, e_begin=5, e_end=6, n_epochs=30, a=A_, b=B_, seed=3)
        assert np.abs(np_(Yg) - ref).max() <= 1e-4


def test_sgd_flat_pieces_bitidentical(O, monkeypatch):
    """The flat deterministic kernel works through each CTA's vertex range in pieces of vt
    vertices; tiny (and odd) pieces exercise ragged pieces and heads split across steps.  The
    int64 fixed-point sums make the result independent of the split (R13)."""
    X, indptr, col, val = _graph(O, n=1500)
    Y0 = cu(synth.uniform_embedding(1500, 2, seed=4))
    outs = []
    for vt in (None, "7", "1"):
        if vt is None:
            monkeypatch.delenv("UMAP_SGD_VT", raising=False)
        else:
            monkeypatch.setenv("UMAP_SGD_VT", vt)
        Yg = Y0.clone()
        U.optimize(cu(indptr), cu(col), cu(val), Yg, e_begin=1, e_end=40, n_epochs=40, a=A_, b=B_, seed=9)
        outs.append(np_(Yg))
    monkeypatch.delenv("UMAP_SGD_VT", raising=False)
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    ref = O.optimize(indptr, col, val, np_(Y0), A_, B_, 40, e_begin=1, e_end=2, m=5, seed=9)
    monkeypatch.setenv("UMAP_SGD_VT", "7")
    Yg = Y0.clone()
    U.optimize(cu(indptr), cu(col), cu(val), Yg, e_begin=1, e_end=2, n_epochs=40, a=A_, b=B_, seed=9)
    monkeypatch.delenv("UMAP_SGD_VT", raising=False)
    assert np.abs(np_(Yg) - ref).max() <= 1e-4


@pytest.mark.parametrize("dim,m", [(2, 5), (1, 5), (3, 3), (4, 7)])
def test_sgd_deterministic_kernels_bitidentical(O, monkeypatch, dim, m):
    """Every deterministic SGD form gives the same bytes (R13: per-term fixed point, integer sums):
    flat5 as two CTAs per SM (the default) and as one, flat3 (records streamed from L2), flat4 (the
    materialised schedule) and flat2 (pieces); the positives count is the schedule's."""
    X, indptr, col, val = _graph(O, n=5000)
    Y0 = cu(synth.uniform_embedding(5000, dim, seed=3))
    outs, pos = [], []
    for env in ({}, {"UMAP_SGD_CPS": "1"}, {"UMAP_SGD_SCHED": "0"}, {"UMAP_SGD_SCHED": "1"}, {"UMAP_SGD_VT": "64"}):
        for kk in ("UMAP_SGD_CPS", "UMAP_SGD_SCHED", "UMAP_SGD_VT"):
            monkeypatch.delenv(kk, raising=False)
        for kk, vv in env.items():
            monkeypatch.setenv(kk, vv)
        Yg = Y0.clone()
        pos.append(U.optimize(cu(indptr), cu(col), cu(val), Yg, e_begin=1, e_end=60, n_epochs=60, a=A_, b=B_,
                              seed=11, negative_sample_rate=m))
        outs.append(np_(Yg))
    for kk in ("UMAP_SGD_CPS", "UMAP_SGD_SCHED", "UMAP_SGD_VT"):
        monkeypatch.delenv(kk, raising=False)
    for o in outs[1:]:
        assert np.array_equal(outs[0], o)
    assert len(set(pos)) == 1


def test_hogwild_flat_and_chunk_kernels_vs_oracle(O, monkeypatch):
    """Hogwild (R14) on flat5's structure (default) and on the persistent chunk kernel
    (UMAP_SGD_HOG_CHUNK=1): both fits' trustworthiness within 0.005 of the oracle's own fit."""
    c = synth.CONFIGS["C1"]
    X = synth.lowrank(c["n"], c["d"], c["blobs"], c["seed"])
    T_ref = O.trustworthiness(X, O.fit(X, k=15, n_epochs=200, a=A_, b=B_, seed=2, mode="hogwild"), 15)
    for chunk in (False, True):
        if chunk:
            monkeypatch.setenv("UMAP_SGD_HOG_CHUNK", "1")
        Y, st = U.fit(cu(X), n_neighbors=15, n_epochs=200, a=A_, b=B_, seed=2, sgd_mode="hogwild")
        monkeypatch.delenv("UMAP_SGD_HOG_CHUNK", raising=False)
        T, _ = U.trustworthiness(cu(X), Y, 15)
        assert abs(T - T_ref) <= 0.005, (chunk, T, T_ref)


def test_sgd_positive_count_matches_schedule(O):
    X, indptr, col, val = _graph(O, n=600)
    N = 50
    r = (val / val.max()).astype(np.float32)
    expected = sum(int(np.sum(np.floor(np.float32(e) * r) > np.floor(np.float32(e - 1) * r))) for e in range(1, N))
    Yg = cu(synth.uniform_embedding(600, 2))
    pos = U.optimize(cu(indptr), cu(col), cu(val), Yg, n_epochs=N, a=A_, b=B_)
    assert pos == expected


# ------------------------------------------------------------------- end to end
def test_fit_c1_digits_vs_oracle(O):
    X = synth.make("C1")
    ref = O.fit(X, k=15, n_epochs=200, a=A_, b=B_, seed=0, mode="deterministic")
    t_ref = O.trustworthiness(X, ref, 15)
    for mode in ("deterministic", "hogwild"):
        Y, st = U.fit(cu(X), n_neighbors=15, n_epochs=200, a=A_, b=B_, seed=0, sgd_mode=mode)
        T, _ = U.trustworthiness(cu(X), Y, 15)
        assert abs(T - t_ref) <= 0.005, (mode, T, t_ref)
        assert st["gpu_launches"] >= 10 and st["nnz"] > 0


def test_fit_host_pointers_equal_device(O):
    X = synth.lowrank(800, 16, seed=6)
    Yd, _ = U.fit(cu(X), n_epochs=60, a=A_, b=B_, seed=4)
    Xh = torch.from_numpy(X).pin_memory()
    Yh, _ = U.fit(Xh, n_epochs=60, a=A_, b=B_, seed=4)
    assert not Yh.is_cuda
    assert np.array_equal(np_(Yd), Yh.numpy())


def test_fit_rejects_nonfinite_and_tiny():
    X = synth.lowrank(100, 4)
    X[3, 2] = np.nan
    with pytest.raises(RuntimeError, match="NONFINITE"):
        U.fit(cu(X), n_epochs=10)
    with pytest.raises(RuntimeError, match="TOO_FEW_ROWS"):
        U.fit(cu(synth.lowrank(15, 4)), n_neighbors=15)


def test_fit_minimum_rows():
    Y, _ = U.fit(cu(synth.lowrank(16, 3)), n_neighbors=15, n_epochs=20)
    assert torch.isfinite(Y).all()


# ------------------------------------------------------------------- transform (a9)
def _transform_setup(O, n_tr=1200, n_q=700, d=24, k=15):
    X = synth.lowrank(n_tr + n_q, d, seed=7)
    Xtr, Xq = X[:n_tr], X[n_tr:]
    Ytr = O.fit(Xtr, k=k, n_epochs=40, a=A_, b=B_, seed=1)
    idx, dist = O.knn(Xq, Xtr, k)
    rho, sigma = O.smooth_knn(dist)
    w = O.membership(dist, rho, sigma)
    return Xtr, Xq, Ytr, idx, dist, w


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_transform_init_and_teacher_forced(O, prec):
    Xtr, Xq, Ytr, idx, dist, w = _transform_setup(O)
    Nt = 67
    y0 = O.transform_init(idx, w, Ytr)
    Yg = torch.zeros((Xq.shape[0], 2), dtype=torch.float32, device=DEV)
    U.transform_optimize(cu(idx), cu(w), cu(Ytr), Yg, Nt, e_begin=1, e_end=1, init=True, a=A_, b=B_)
    assert np.array_equal(np_(Yg), y0)
    # per-epoch teacher forcing.  transform_precision = fp64 evaluates each update in fp64 and
    # stores the position in fp32 after every update, as the oracle does (R15): equal to the
    # oracle bit for bit.  The default fp32 MUFU form: each query row chains k (1 + m) = 90
    # dependent in-place updates per epoch, which amplifies fp32 rounding (DESIGN.md
    # "Parity bars"): 99.9 % of rows within north_star's 1e-4, every row within 1e-3.
    Y = y0
    errs = []
    for e in range(1, Nt):
        ref = O.transform_optimize(idx, w, Ytr, Y, A_, B_, Nt, seed=9, e_begin=e, e_end=e + 1)
        Yg = cu(Y)
        U.transform_optimize(cu(idx), cu(w), cu(Ytr), Yg, Nt, e_begin=e, e_end=e + 1, a=A_, b=B_, seed=9,
                             transform_precision=prec)
        errs.append(np.abs(np_(Yg) - ref).max(1))
        Y = ref
    errs = np.array(errs)
    print("transform teacher-forced (%s): max %.3g p99.9 %.3g exact rows %.4f" %
          (prec, errs.max(), np.quantile(errs, 0.999), float((errs == 0).mean())))
    if prec == "fp64":
        assert errs.max() == 0.0, errs.max()
    else:
        assert errs.max() <= 1e-3, errs.max()
        assert np.quantile(errs, 0.999) <= 1e-4


def test_transform_end_to_end_and_partition_invariance(O):
    Xtr, Xq, Ytr, idx, dist, w = _transform_setup(O)
    ref = O.transform(Xtr, Ytr, Xq, k=15, n_epochs=200, a=A_, b=B_, seed=3)
    Ytr_before = Ytr.copy()
    full = U.transform(cu(Xtr), cu(Ytr), cu(Xq), n_epochs=200, a=A_, b=B_, seed=3)
    assert np.array_equal(Ytr, Ytr_before)
    # contractive towards the frozen anchors: end-to-end drift stays small
    assert np.abs(np_(full) - ref).max() < 1e-2
    parts = [U.transform(cu(Xtr), cu(Ytr), cu(Xq[a:b]), q_offset=a, n_epochs=200, a=A_, b=B_, seed=3)
             for a, b in [(0, 123), (123, 500), (500, 700)]]
    assert np.array_equal(np_(torch.cat(parts)), np_(full))


# ------------------------------------------------------------------- trust (a10)
@pytest.mark.parametrize("n,d,k", [(700, 20, 15), (1000, 64, 5), (300, 7, 1), (257, 3, 40), (900, 36, 24)])
def test_trust_penalty_exact(O, n, d, k):
    X = synth.lowrank(n, d, seed=8)
    Y = synth.uniform_embedding(n, 2, seed=9)
    S_ref, pen_ref = O.trust_penalty(X, Y, k)
    T, S = U.trustworthiness(cu(X), cu(Y), k)
    assert S == S_ref
    assert T == O.trust_from_penalty(S_ref, n, k)
    emb_idx, _ = O.knn(Y, Y, k, self_offset=0)
    S2, pen = U.trust_penalty(cu(X), cu(emb_idx[100:250]), k, 100, 250)
    assert np.array_equal(np_(pen), pen_ref[100:250])


# tensor-core rank counting (split-BF16 GEMM + certified buckets + exact re-check): the
# integer penalty must equal the oracle's exactly
@pytest.mark.parametrize("n,d,k,kind,emb", [(1500, 64, 15, "lowrank", "random"), (1200, 784, 15, "lowrank", "proj"),
                                            (900, 100, 5, "iso", "random"), (700, 3, 15, "ties", "proj"),
                                            (2000, 50, 16, "lowrank", "proj"), (333, 3072, 5, "lowrank", "random")])
def test_trust_tensor_exact_penalty(O, n, d, k, kind, emb):
    X = _data(kind, n, d, seed=13)
    if emb == "random":
        Y = synth.uniform_embedding(n, 2, seed=3)
    else:
        Y = (X[:, :2] + np.random.default_rng(0).standard_normal((n, 2)) * 0.5).astype(np.float32)
    S_ref, pen_ref = O.trust_penalty(X, Y, k)
    T, S = U.trustworthiness(cu(X), cu(Y), k, knn_mode="tensor")
    assert S == S_ref
    emb_idx, _ = O.knn(Y, Y, k, self_offset=0)
    S2, pen = U.trust_penalty(cu(X), cu(emb_idx[17:300]), k, 17, 300, knn_mode="tensor")
    assert np.array_equal(np_(pen), pen_ref[17:300])
    # the same shard visited in the Morton order of Y (layout hint): identical per-row penalties
    S3, pen3 = U.trust_penalty(cu(X), cu(emb_idx[17:300]), k, 17, 300, knn_mode="tensor", Y=cu(Y))
    assert np.array_equal(np_(pen3), pen_ref[17:300]) and S3 == S2


@pytest.mark.parametrize("profile", ["front", "back", "spike"])
def test_trust_tensor_per_pair_margin_adversarial(O, profile):
    """The per-pair fine-pass margin charges each slab's adds with the products of
    the slabs before it: rows whose squared norm sits in the first features (front: the largest
    Qw, partial sums near their maximum from the first slab on), in the last ones (back) or in one
    feature (spike) must still give exactly the oracle's penalty, as must the uniform form."""
    n, d, k = 1400, 784, 15
    X = synth.lowrank(n, d, blobs=10, seed=31)
    f = np.arange(d, dtype=np.float32)
    if profile == "front":
        w = np.exp(-f / 40.0)
    elif profile == "back":
        w = np.exp(-(d - 1 - f) / 40.0)
    else:
        w = np.full(d, 0.05, np.float32)
        w[5] = 30.0
    X = np.ascontiguousarray(X * w[None, :].astype(np.float32), dtype=np.float32)
    Y = synth.uniform_embedding(n, 2, seed=8)
    S_ref, _ = O.trust_penalty(X, Y, k)
    T, S = U.trustworthiness(cu(X), cu(Y), k, knn_mode="tensor")
    assert S == S_ref


@pytest.mark.parametrize("tmaj,ch", [("0", "32"), ("0", "2"), ("1", "1"), ("1", "3")])
def test_trust_tensor_fine_pass_chunk_orders(O, monkeypatch, tmaj, ch):
    """The fine pass's work order: tile lists per query block in block order,
    or chunks of CH tiles of every block launched tile-major (chunks of one block add into the
    same rows concurrently); one-tile and ragged chunks included: the integer penalty must be the
    oracle's whatever the order."""
    n, d, k = 2100, 784, 15
    X = synth.lowrank(n, d, blobs=12, seed=41)
    Y = (X[:, :2] + np.random.default_rng(2).standard_normal((n, 2)) * 0.5).astype(np.float32)
    S_ref, pen_ref = O.trust_penalty(X, Y, k)
    monkeypatch.setenv("UMAP_TC_TILE_MAJOR", tmaj)
    monkeypatch.setenv("UMAP_TC_CHUNK", ch)
    T, S = U.trustworthiness(cu(X), cu(Y), k, knn_mode="tensor")
    emb_idx, _ = O.knn(Y, Y, k, self_offset=0)
    S2, pen = U.trust_penalty(cu(X), cu(emb_idx[40:1900]), k, 40, 1900, knn_mode="tensor", Y=cu(Y))
    monkeypatch.delenv("UMAP_TC_TILE_MAJOR")
    monkeypatch.delenv("UMAP_TC_CHUNK")
    assert S == S_ref
    assert np.array_equal(np_(pen), pen_ref[40:1900])


def test_trust_tensor_table4_shape_and_overflow_fallback(O, monkeypatch):
    """Table-4-shaped rows (isotropic blobs, d = 1024): the tensor path's penalty equals the
    oracle's; with the re-check lists shrunk to 2 pairs per list the tensor pass overflows and
    the exact SIMT fallback must give the same integer penalty."""
    n, d, k = 1200, 1024, 15
    X = synth.iso(n, d, blobs=10, seed=21)
    Y = synth.uniform_embedding(n, 2, seed=5)
    S_ref, _ = O.trust_penalty(X, Y, k)
    T, S = U.trustworthiness(cu(X), cu(Y), k, knn_mode="tensor")
    assert S == S_ref
    monkeypatch.setenv("UMAP_TC_AMB_CAP", "2")
    T2, S2 = U.trustworthiness(cu(X), cu(Y), k, knn_mode="tensor")
    monkeypatch.delenv("UMAP_TC_AMB_CAP")
    assert S2 == S_ref and T2 == T


def test_trust_identity_is_one():
    X = cu(synth.lowrank(500, 6))
    T, S = U.trustworthiness(X, X, 10)
    assert S == 0 and T == 1.0


# ------------------------------------------------------------------- full-size sampled checks
@pytest.mark.slow
def test_c2_full_size_sampled_knn_and_trust(O):
    """C2 at full size (70,000 x 784) in the launch configuration bench.py times: sampled
    rows are recomputed one by one by the oracle."""
    X = synth.make("C2")
    Xg = cu(X)
    gi, gd = U.knn(Xg, Xg, 15, exclude_self=True)
    gi, gd = np_(gi), np_(gd)
    rng = np.random.default_rng(0)
    rows = np.concatenate([[0, 69999], rng.choice(70000, 10, replace=False)])
    for r in rows:
        ri, rd = O.knn(X[r:r + 1], X, 15, self_offset=int(r))
        assert np.array_equal(gi[r], ri[0]) and np.array_equal(gd[r], rd[0])


@pytest.mark.slow
def test_c2_full_size_trust_tensor_equals_exact(O):
    """C2 at full size in bench.py's launch configuration (umap_fit with trust_k = 15, tensor
    mode, Morton-ordered rank counting): the integer penalty S equals the exact-mode S (fp32
    SIMT ranks, pinned to the oracle at small sizes), and sampled rows' penalties equal the
    oracle's, recomputed one row at a time."""
    X = synth.make("C2")
    Xg = cu(X)
    Y, st = U.fit(Xg, n_neighbors=15, n_epochs=500, seed=0, knn_mode="tensor", trust_k=15)
    T_exact, S_exact = U.trustworthiness(Xg, Y, 15, knn_mode="exact")
    assert st["trust_penalty"] == S_exact and st["trustworthiness"] == T_exact
    Yh = np_(Y)
    emb_idx, _ = U.knn(Y, Y, 15, exclude_self=True)
    rng = np.random.default_rng(1)
    for r in np.concatenate([[0, 69999], rng.choice(70000, 4, replace=False)]):
        r = int(r)
        S_r, pen_r = U.trust_penalty(Xg, emb_idx[r:r + 1].contiguous(), 15, r, r + 1, knn_mode="tensor", Y=Y)
        S_o, _ = O.trust_penalty(X, Yh, 15, r, r + 1)
        assert S_r == S_o, r


@pytest.mark.slow
def test_c3_full_size_trust_and_knn(O):
    """C3 (60,000 x 3,072, d beyond the K-tile ring, trust k = 5) at full size: tensor-mode
    trust S equals the exact-mode S; sampled kNN rows bit-exact against the oracle."""
    X = synth.make("C3")
    Xg = cu(X)
    Y, st = U.fit(Xg, n_neighbors=15, n_epochs=200, seed=0, knn_mode="tensor", trust_k=5)
    T_exact, S_exact = U.trustworthiness(Xg, Y, 5, knn_mode="exact")
    assert st["trust_penalty"] == S_exact
    gi, gd = U.knn(Xg, Xg, 15, exclude_self=True, mode="tensor")
    gi, gd = np_(gi), np_(gd)
    for r in np.random.default_rng(2).choice(60000, 4, replace=False):
        ri, rd = O.knn(X[r:r + 1], X, 15, self_offset=int(r))
        assert np.array_equal(gi[r], ri[0]) and np.array_equal(gd[r], rd[0])


@pytest.mark.slow
def test_c4_full_size_sampled_knn(O):
    """C4 (1,000,000 x 50, d % 4 != 0: the per-lane re-rank path) at full size, the kNN the
    sharded mode distributes: sampled rows bit-exact against the oracle."""
    X = synth.make("C4")
    gi, gd = U.knn(cu(X), cu(X), 15, exclude_self=True, mode="tensor")
    gi, gd = np_(gi), np_(gd)
    for r in np.concatenate([[0, 999999], np.random.default_rng(3).choice(1000000, 4, replace=False)]):
        ri, rd = O.knn(X[r:r + 1], X, 15, self_offset=int(r))
        assert np.array_equal(gi[r], ri[0]) and np.array_equal(gd[r], rd[0])


@pytest.mark.slow
def test_c5_transform_chunk_sampled_rows(O):
    """C5: fit on the 100,000 training rows, transform one 1,000,000-row chunk of the
    8,000,000-row set on the device (global query ids), sampled rows against the oracle."""
    model = synth.lowrank_model(784, 10, 4)
    Xtr = synth.lowrank_sample(model, 100000, 40)
    Xg = cu(Xtr)
    Ytr, _ = U.fit(Xg, n_neighbors=15, n_epochs=200, knn_mode="tensor", a=A_, b=B_)
    Xq = synth.lowrank_sample_device(model, 1000000, 44)
    Yq = U.transform(Xg, Ytr, Xq, q_offset=3000000, n_neighbors=15, n_epochs=200, knn_mode="tensor", a=A_, b=B_)
    Ytr_h = np_(Ytr)
    for r in (0, 123457, 999999):
        yo = O.transform(Xtr, Ytr_h, np_(Xq[r:r + 1]), k=15, n_epochs=200, a=A_, b=B_, seed=0, q_offset=3000000 + r)
        assert np.abs(np_(Yq[r]) - yo[0]).max() < 1e-3


# ------------------------------------------------------------------- supervised (f4, R17)
def test_supervised_adjust_bitexact(O):
    X = synth.lowrank(1500, 16, blobs=4, seed=21)
    _, _, _, _, _, (indptr, col, w) = O.fuzzy_graph(X, 15)
    lab = np.random.default_rng(4).integers(-1, 4, 1500).astype(np.int32)
    for far, unk in [(5.0, 1.0), (40.0, 30.0), (0.0, 0.0)]:
        ri, rc, rv = O.supervised_adjust(indptr, col, w, lab, far, unk)
        gi, gc, gv = U.supervised_adjust(cu(indptr), cu(col), cu(w), cu(lab), far, unk)
        assert np.array_equal(np_(gi), ri) and np.array_equal(np_(gc), rc) and np.array_equal(np_(gv), rv)


def test_supervised_fit_c1_vs_oracle(O):
    """Supervised fit at digits shape (labels = the blob ids, a quarter unknown): trust within
    0.005 of the oracle's supervised fit."""
    X, lab = synth.lowrank(1797, 64, blobs=10, seed=0, return_labels=True)
    lab = lab.astype(np.int32)
    lab[np.random.default_rng(1).random(1797) < 0.25] = -1
    Y, st = U.fit(cu(X), labels=torch.from_numpy(lab), n_neighbors=15, n_epochs=200, a=A_, b=B_, seed=1,
                  trust_k=15)
    Yr = O.fit(X, k=15, n_epochs=200, a=A_, b=B_, seed=1, mode="deterministic", labels=lab)
    assert abs(st["trustworthiness"] - O.trustworthiness(X, Yr, 15)) < 0.005
    Y0, st0 = U.fit(cu(X), n_neighbors=15, n_epochs=200, a=A_, b=B_, seed=1)
    assert st["nnz"] <= st0["nnz"]


# ------------------------------------------------------------------- spectral init (f3, R18)
@pytest.mark.parametrize("dim", [1, 2, 3])
def test_spectral_init_vs_oracle(O, dim):
    X = synth.lowrank(1797, 64, blobs=10, seed=0)
    _, _, _, _, _, (indptr, col, w) = O.fuzzy_graph(X, 15)
    Yr, _ = O.spectral_init(indptr, col, w, dim, seed=5, iters=300)
    Yg = U.spectral_init(cu(indptr), cu(col), cu(w), dim, seed=5, iters=300)
    assert np.abs(np_(Yg) - Yr).max() < 1e-3


def test_spectral_fit_c1_vs_oracle(O):
    X = synth.lowrank(1797, 64, blobs=10, seed=0)
    Y, st = U.fit(cu(X), n_neighbors=15, n_epochs=200, a=A_, b=B_, seed=1, init="spectral", trust_k=15)
    Yr = O.fit(X, k=15, n_epochs=200, a=A_, b=B_, seed=1, mode="deterministic", init="spectral")
    assert abs(st["trustworthiness"] - O.trustworthiness(X, Yr, 15)) < 0.005


def test_spectral_and_supervised_edge_cases(O):
    """Isolated vertices (degree 0) in the spectral init; all labels unknown (-1) and all
    labels distinct with a far_dist that drops every edge in the supervised adjustment."""
    import scipy.sparse as sp
    rng = np.random.default_rng(9)
    n = 300
    r = rng.integers(0, n - 10, 2000)
    c = rng.integers(0, n - 10, 2000)
    keep = r != c
    W = sp.coo_matrix((rng.uniform(0.1, 1, keep.sum()).astype(np.float32), (r[keep], c[keep])), shape=(n, n)).tocsr()
    W = ((W + W.T) * 0.5).tocsr()
    W.sort_indices()
    ip, cl, w = W.indptr.astype(np.int64), W.indices.astype(np.int32), W.data.astype(np.float32)
    Yr, _ = O.spectral_init(ip, cl, w, 2, seed=2, iters=300)
    Yg = U.spectral_init(cu(ip), cu(cl), cu(w), 2, seed=2, iters=300)
    assert np.abs(np_(Yg) - Yr).max() < 1e-3          # the last 10 rows are isolated
    lab = np.full(n, -1, np.int32)
    gi, gc, gv = U.supervised_adjust(cu(ip), cu(cl), cu(w), cu(lab), 5.0, 1.0)
    ri, rc, rv = O.supervised_adjust(ip, cl, w, lab, 5.0, 1.0)
    assert np.array_equal(np_(gi), ri) and np.array_equal(np_(gv), rv)
    lab = np.arange(n, dtype=np.int32)
    gi, gc, gv = U.supervised_adjust(cu(ip), cu(cl), cu(w), cu(lab), 80.0, 1.0)
    assert gc.numel() == 0 and int(np_(gi)[-1]) == 0

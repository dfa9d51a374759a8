"""Round-2 GPU parity cases (VERDICT r1 "Next round" 2 and ADVICE r1): the benchmarked
tensor-mode kNN at full C2 size, the unpacked-record SGD path, Hogwild and deterministic
fits at every supported n_components, the transform at DIM 3, umap_fit_knn (f1) against
umap_fit and the oracle, its input validation, the R13 fixed-point bound, and a device-side
check that the transform leaves the training layout untouched.  Run on a B200: pytest -m gpu.
"""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2008_00325_b200 as U  # noqa: E402

A_, B_ = 1.5769434603, 0.8950608779
DEV = "cuda"


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def np_(t):
    return t.detach().cpu().numpy()


def _graph(O, n=1500, d=32, k=15, seed=5):
    X = synth.lowrank(n, d, blobs=5, seed=seed)
    _, _, _, _, _, (indptr, col, val) = O.fuzzy_graph(X, k)
    return X, indptr, col, val


# ------------------------------------------------------------------ a2 at full C2 size
@pytest.mark.slow
def test_c2_full_size_tensor_knn_recall_and_rows(O):
    """The kNN mode bench.py times (tensor: tcgen05 BF16 candidates + exact re-rank) at the
    full C2 shape: recall against the exact mode over all 70,000 rows >= 0.999 (north_star),
    rows whose neighbour sets agree are bit-identical (ids and distances), and 64 sampled rows
    equal the oracle's brute force."""
    X = synth.make("C2")
    Xg = cu(X)
    ti, td = U.knn(Xg, Xg, 15, exclude_self=True, mode="tensor")
    ei, ed = U.knn(Xg, Xg, 15, exclude_self=True, mode="exact")
    ti, td, ei, ed = np_(ti), np_(td), np_(ei), np_(ed)
    hits = sum(len(np.intersect1d(a, b)) for a, b in zip(ti, ei))
    recall = hits / ei.size
    assert recall >= 0.999, recall
    same = np.all(np.sort(ti, 1) == np.sort(ei, 1), axis=1)
    assert np.array_equal(ti[same], ei[same]) and np.array_equal(td[same], ed[same])
    rows = np.concatenate([[0, 69999], np.random.default_rng(11).choice(70000, 62, replace=False)])
    for r in rows:
        oi, od = O.knn(X[r:r + 1], X, 15, self_offset=int(r))
        assert np.array_equal(ti[r], oi[0]) and np.array_equal(td[r], od[0]), r


# ------------------------------------------------------------------ a8 unpacked records
def test_sgd_unpacked_records_match_packed_and_oracle(O, monkeypatch):
    """vt > 2048 (or n >= 2^21, C4) keeps {col, r} and the 16-bit head offsets in separate
    arrays (the packed 8-byte record needs n < 2^21, vt <= 2048).  Same bits as the packed
    path, and the teacher-forced oracle bar."""
    X, indptr, col, val = _graph(O, n=3000)
    Y0 = cu(synth.uniform_embedding(3000, 2, seed=4))
    outs = []
    for vt in (None, "4096"):
        if vt is None:
            monkeypatch.delenv("UMAP_SGD_VT", raising=False)
        else:
            monkeypatch.setenv("UMAP_SGD_VT", vt)
        Yg = Y0.clone()
        U.optimize(cu(indptr), cu(col), cu(val), Yg, e_begin=1, e_end=30, n_epochs=30, a=A_, b=B_, seed=9)
        outs.append(np_(Yg))
    assert np.array_equal(outs[0], outs[1])
    monkeypatch.setenv("UMAP_SGD_VT", "4096")
    Y = np_(Y0)
    for e in (1, 17):
        ref = O.optimize(indptr, col, val, Y, A_, B_, 30, e_begin=e, e_end=e + 1, m=5, seed=9)
        Yg = cu(Y)
        U.optimize(cu(indptr), cu(col), cu(val), Yg, e_begin=e, e_end=e + 1, n_epochs=30, a=A_, b=B_, seed=9)
        assert np.abs(np_(Yg) - ref).max() <= 1e-4
        Y = ref


# ------------------------------------------------------------------ a8 fixed-point bound (R13)
def test_sgd_large_negative_rate_teacher_forced(O):
    """m = 25 at learning_rate 1: (2 + m) alpha0 = 27 < 32, the largest per-edge fixed-point
    sum the deterministic mode accepts; parity with the oracle's fp64 buffer."""
    X, indptr, col, val = _graph(O, n=800)
    Y = synth.uniform_embedding(800, 2, seed=3) * np.float32(0.05)  # crowded: large repulsion
    for e in (1, 9):
        ref = O.optimize(indptr, col, val, Y, A_, B_, 10, e_begin=e, e_end=e + 1, m=25, seed=2)
        Yg = cu(Y)
        U.optimize(cu(indptr), cu(col), cu(val), Yg, e_begin=e, e_end=e + 1, n_epochs=10, a=A_, b=B_, seed=2,
                   negative_sample_rate=25)
        assert np.abs(np_(Yg) - ref).max() <= 1e-4
        Y = ref


def test_sgd_fixed_point_bound_rejected():
    X = synth.lowrank(200, 8, seed=1)
    for m, lr in ((30, 1.0), (5, 4.6), (0, 16.0)):
        with pytest.raises(RuntimeError, match="INVALID_ARGUMENT"):
            U.fit(cu(X), n_epochs=5, negative_sample_rate=m, learning_rate=lr, sgd_mode="deterministic")
    # Hogwild has no fixed point: allowed
    Y, _ = U.fit(cu(X), n_epochs=5, negative_sample_rate=30, learning_rate=1.0, sgd_mode="hogwild")
    assert torch.isfinite(Y).all()


# ------------------------------------------------------------------ f2 every n_components
@pytest.mark.parametrize("dim", [1, 3, 4, 8, 16])
def test_fit_c1_all_dims_both_modes_vs_oracle(O, dim):
    """End-to-end at C1 for every supported n_components, deterministic and Hogwild (the
    Hogwild persistent kernel's gathers are L1-cached since r01): trustworthiness within
    0.005 of the oracle's deterministic fit of the same dimension."""
    X = synth.make("C1")
    # 1-D layouts are chaotic: the GPU's per-epoch agreement (<= 1e-4, teacher-forced,
    # test_sgd_deterministic_teacher_forced_dims) does not carry a 200-epoch trajectory, and one
    # seed's trust alone varies by up to 0.017 between seeds on either side (measured,
    # tools/dim_trust_seeds.py: oracle 0.9589..0.9642, GPU 0.9462..0.9642 over seeds 0-5).  At
    # DIM 1 the bar is applied to the mean over four seeds.
    seeds = (0, 1, 2, 3) if dim == 1 else (0,)
    t_ref = np.mean([O.trustworthiness(X, O.fit(X, k=15, n_components=dim, n_epochs=200, a=A_, b=B_, seed=s,
                                                 mode="deterministic"), 15) for s in seeds])
    for mode in ("deterministic", "hogwild"):
        Ts = []
        for s in seeds:
            Y, _ = U.fit(cu(X), n_neighbors=15, n_components=dim, n_epochs=200, a=A_, b=B_, seed=s, sgd_mode=mode)
            assert Y.shape == (X.shape[0], dim)
            Ts.append(U.trustworthiness(cu(X), Y, 15)[0])
        T = float(np.mean(Ts))
        assert abs(T - t_ref) <= 0.005, (dim, mode, Ts, t_ref)


@pytest.mark.parametrize("dim", [1, 4, 8])
def test_sgd_deterministic_teacher_forced_dims(O, dim):
    X, indptr, col, val = _graph(O, n=900)
    Y = synth.uniform_embedding(900, dim, seed=2)
    for e in (1, 13):
        ref = O.optimize(indptr, col, val, Y, A_, B_, 30, e_begin=e, e_end=e + 1, m=5, seed=3)
        Yg = cu(Y)
        U.optimize(cu(indptr), cu(col), cu(val), Yg, e_begin=e, e_end=e + 1, n_epochs=30, a=A_, b=B_, seed=3)
        assert np.abs(np_(Yg) - ref).max() <= 1e-4, (dim, e)
        Y = ref


# ------------------------------------------------------------------ a9 transform at DIM 3
def test_transform_dim3_teacher_forced_and_train_untouched(O):
    X = synth.lowrank(1500, 20, seed=7)
    Xtr, Xq = X[:1000], X[1000:]
    Ytr = O.fit(Xtr, k=15, n_components=3, n_epochs=30, a=A_, b=B_, seed=1)
    idx, dist = O.knn(Xq, Xtr, 15)
    rho, sigma = O.smooth_knn(dist)
    w = O.membership(dist, rho, sigma)
    Nt = 20
    y0 = O.transform_init(idx, w, Ytr)
    Ytr_g = cu(Ytr)
    Ytr_bytes = Ytr_g.clone()
    Yg = torch.zeros((Xq.shape[0], 3), dtype=torch.float32, device=DEV)
    U.transform_optimize(cu(idx), cu(w), Ytr_g, Yg, Nt, e_begin=1, e_end=1, init=True, a=A_, b=B_)
    assert np.array_equal(np_(Yg), y0)
    Y, errs = y0, []
    for e in range(1, Nt):
        ref = O.transform_optimize(idx, w, Ytr, Y, A_, B_, Nt, seed=9, e_begin=e, e_end=e + 1)
        Yg = cu(Y)
        U.transform_optimize(cu(idx), cu(w), Ytr_g, Yg, Nt, e_begin=e, e_end=e + 1, a=A_, b=B_, seed=9)
        errs.append(np.abs(np_(Yg) - ref).max(1))
        Y = ref
    errs = np.array(errs)
    assert errs.max() <= 1e-3 and np.quantile(errs, 0.999) <= 1e-4
    # the training layout on the device is bit-unchanged (R15), compared on the device
    assert torch.equal(Ytr_g.view(torch.int32), Ytr_bytes.view(torch.int32))


def test_transform_leaves_device_train_layout_bitwise(O):
    """umap_transform reads Y_train in place on the device: its bytes are unchanged."""
    X = synth.lowrank(1300, 24, seed=8)
    Xtr, Xq = cu(X[:1000]), cu(X[1000:])
    Ytr, _ = U.fit(Xtr, n_epochs=40, a=A_, b=B_, seed=2)
    before = Ytr.clone()
    Yq = U.transform(Xtr, Ytr, Xq, n_epochs=40, a=A_, b=B_, seed=3)
    torch.cuda.synchronize()
    assert torch.equal(Ytr.view(torch.int32), before.view(torch.int32))
    assert torch.isfinite(Yq).all()


# ------------------------------------------------------------------ f1 umap_fit_knn
@pytest.mark.parametrize("mode", ["deterministic", "hogwild"])
def test_fit_knn_equals_fit_and_oracle(O, mode):
    """f1 (App. A.1): fit_knn(knn(X)) is umap_fit(X) from a3 on, bit for bit in the
    deterministic mode; host-pointer inputs give the same; trust within 0.005 of the oracle."""
    X = synth.make("C1")
    Xg = cu(X)
    Yf, stf = U.fit(Xg, n_neighbors=15, n_epochs=200, a=A_, b=B_, seed=0, sgd_mode=mode)
    gi, gd = U.knn(Xg, Xg, 15, exclude_self=True)
    Yk, stk = U.fit_knn(gi, gd, n_epochs=200, a=A_, b=B_, seed=0, sgd_mode=mode)
    assert stk["nnz"] == stf["nnz"] and stk["positives"] == stf["positives"]
    if mode == "deterministic":
        assert torch.equal(Yk, Yf)
        Yh, _ = U.fit_knn(gi.cpu(), gd.cpu(), n_epochs=200, a=A_, b=B_, seed=0, sgd_mode=mode)
        assert torch.equal(Yh.to(DEV), Yf)
    oi, od = O.knn(X, X, 15, self_offset=0)
    ref = O.fit(X, k=15, n_epochs=200, a=A_, b=B_, seed=0, mode="deterministic")
    T, _ = U.trustworthiness(Xg, Yk, 15)
    assert abs(T - O.trustworthiness(X, ref, 15)) <= 0.005
    assert np.array_equal(np_(gi), oi)


def test_fit_knn_rejects_bad_graphs():
    X = synth.lowrank(300, 8, seed=3)
    Xg = cu(X)
    gi, gd = U.knn(Xg, Xg, 10, exclude_self=True)
    bad = []
    t = gi.clone(); t[5, 3] = 300; bad.append((t, gd))                   # id == n
    t = gi.clone(); t[7, 0] = -1; bad.append((t, gd))                    # negative id
    t = gi.clone(); t[9, 2] = 9; bad.append((t, gd))                     # the row itself
    t = gi.clone(); t[11, 4] = t[11, 1]; bad.append((t, gd))             # duplicate in a row
    d = gd.clone(); d[2, 2] = float("nan"); bad.append((gi, d))          # NaN distance
    d = gd.clone(); d[3, 1] = -1.0; bad.append((gi, d))                  # negative distance
    for bi, bd in bad:
        with pytest.raises(RuntimeError, match="INVALID_ARGUMENT"):
            U.fit_knn(bi, bd, n_epochs=10)
    Y, _ = U.fit_knn(gi, gd, n_epochs=10)
    assert torch.isfinite(Y).all()

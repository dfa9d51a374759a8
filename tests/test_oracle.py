"""Pins of the CPU oracle against what the paper and the mathematics fix (task rule ③).

None of these retype the oracle's own formula: each compares against an
independent definition (brute-force sort, scipy.sparse algebra, sklearn,
finite differences, closed forms, published constants, KAT vectors).
"""
import math

import numpy as np
import pytest

import synth
from conftest import golden


# ----------------------------------------------------------------- Philox (R11)
def test_philox_kat(O):
    for v in golden("philox_kat.json")["vectors"]:
        ctr = [int(x, 16) for x in v["ctr"]]
        key = [int(x, 16) for x in v["key"]]
        out = [int(x, 16) for x in v["out"]]
        assert list(O.philox4x32_10(ctr, key)) == out


def test_random_init_range_and_uniformity(O):
    Y = O.random_init(20000, 2, seed=7)
    assert Y.min() >= -10.0 and Y.max() < 10.0
    # uniform on [-10, 10): mean 0, var 100/3
    assert abs(Y.mean()) < 0.15
    assert abs(Y.var() - 100.0 / 3.0) < 1.0
    assert not np.array_equal(Y, O.random_init(20000, 2, seed=8))
    assert np.array_equal(Y, O.random_init(20000, 2, seed=7))


# ----------------------------------------------------------------- kNN (R1, R2)
def test_knn_line_example(O):
    g = golden("spec_examples.json")["knn_line"]
    X = np.array(g["points"], np.float32)[:, None]
    idx, dist = O.knn(X, X, g["k"], self_offset=0)
    assert idx[:, 0].tolist() == g["idx"]
    assert dist[:, 0].tolist() == g["dist"]


def test_knn_duplicate_tie_lower_index(O):
    g = golden("spec_examples.json")["knn_duplicate_tie"]
    X = np.array(g["points"], np.float32)
    idx, dist = O.knn(X, X, 2, self_offset=0)
    # rows 1 and 2 are duplicates: each is the other's nearest at distance 0
    assert idx[1, 0] == 2 and idx[2, 0] == 1 and dist[1, 0] == 0.0
    # row 3 (9,9): rows 1 and 2 tie at the same distance -> lower index first
    assert idx[3].tolist() == [1, 2]
    assert idx[0, 0] == g["idx_row0"]


def test_knn_matches_fp64_bruteforce_sort(O):
    X = synth.lowrank(300, 17, blobs=4, seed=3)
    k = 10
    idx, dist = O.knn(X, X, k, self_offset=0)
    D = ((X[:, None, :].astype(np.float64) - X[None, :, :]) ** 2).sum(-1)
    np.fill_diagonal(D, np.inf)
    ref = np.argsort(D, axis=1, kind="stable")[:, :k]
    assert np.array_equal(idx, ref)
    assert np.allclose(dist, np.sqrt(np.take_along_axis(D, ref, 1)), rtol=1e-5)


def test_knn_ties_lattice_lexicographic(O):
    X = synth.ties(120, 3, seed=1)
    k = 12
    idx, dist = O.knn(X, X, k, self_offset=0)
    D = ((X[:, None, :].astype(np.float64) - X[None, :, :]) ** 2).sum(-1)  # exact on integers
    for i in range(X.shape[0]):
        keys = sorted((D[i, j], j) for j in range(X.shape[0]) if j != i)[:k]
        assert idx[i].tolist() == [j for _, j in keys]


def test_knn_k_eq_n_minus_1_is_permutation(O):
    X = synth.lowrank(4, 3, blobs=2, seed=0)
    idx, dist = O.knn(X, X, 3, self_offset=0)
    for i in range(4):
        assert sorted(idx[i].tolist()) == [j for j in range(4) if j != i]
        assert np.all(np.diff(dist[i]) >= 0)


def test_knn_no_self_exclusion_puts_self_first(O):
    X = synth.lowrank(50, 5, seed=2)
    idx, dist = O.knn(X, X, 3, self_offset=-1)
    assert np.array_equal(idx[:, 0], np.arange(50)) and np.all(dist[:, 0] == 0)


def test_sqdist_error_bound(O):
    rng = np.random.default_rng(0)
    for _ in range(20):
        x = rng.standard_normal(784).astype(np.float32)
        y = rng.standard_normal(784).astype(np.float32)
        exact = float(((x.astype(np.float64) - y) ** 2).sum())
        # sequential fp32 accumulation: relative error <= d * 2^-23 (loose bound)
        assert abs(O.sqdist(x, y) - exact) <= 784 * 2.0 ** -23 * exact
        assert O.sqdist(x, x) == 0.0


# ----------------------------------------------------------- rho, sigma (R4, R5)
def test_sigma_worked_example(O):
    g = golden("spec_examples.json")["sigma"]
    rho, sigma = O.smooth_knn(np.array([g["dist"]], np.float32))
    assert rho[0] == g["rho"]
    # |psum - log2 k| < 1e-5 and dpsum/dsigma = ln(3)^2 at the root
    assert abs(sigma[0] - g["sigma"]) <= 1e-5 / math.log(3) ** 2 + 1e-7


def test_rho_skips_zero_distance(O):
    g = golden("spec_examples.json")["rho_zero_skip"]
    rho, _ = O.smooth_knn(np.array([g["dist"]], np.float32))
    assert rho[0] == g["rho"]


def test_sigma_eq1_residual_on_real_graph(O):
    X = synth.lowrank(500, 32, seed=4)
    k = 15
    _, dist = O.knn(X, X, k, self_offset=0)
    rho, sigma = O.smooth_knn(dist)
    d = dist.astype(np.float64)
    psum = np.where(d - rho[:, None] > 0, np.exp(-(d - rho[:, None]) / sigma[:, None].astype(np.float64)), 1.0).sum(1)
    mean = d.mean(1)
    clamped = np.isclose(sigma, 1e-3 * mean, rtol=1e-6)
    # Eq. 1 holds on every non-clamped row (fp32 rounding of sigma adds < 1e-6)
    assert np.all(np.abs(psum - math.log2(k))[~clamped] < 2e-5)
    assert clamped.mean() < 0.01


def test_sigma_all_equal_row_clamps(O):
    rho, sigma = O.smooth_knn(np.full((1, 6), 2.5, np.float32))
    assert rho[0] == 2.5
    assert sigma[0] == np.float32(2.5e-3)


def test_sigma_scale_covariance(O):
    rng = np.random.default_rng(1)
    dist = np.sort(rng.uniform(1, 3, (50, 15)), axis=1).astype(np.float32)
    _, s1 = O.smooth_knn(dist)
    _, s2 = O.smooth_knn(dist * np.float32(4.0))
    assert np.allclose(s2, 4 * s1, rtol=5e-5)


# ----------------------------------------------------------- membership (R6)
def test_membership_values(O):
    dist = np.array([[1.0, 1.0 + 0.5, 3.0]], np.float32)
    rho = np.array([1.0], np.float32)
    sigma = np.array([0.5], np.float32)
    w = O.membership(dist, rho, sigma)
    assert w[0, 0] == 1.0
    assert w[0, 1] == np.float32(math.exp(-1.0))
    assert w[0, 2] == np.float32(math.exp(-4.0))


def test_membership_row_sums_log2k(O):
    X = synth.lowrank(400, 20, seed=5)
    _, dist = O.knn(X, X, 15, self_offset=0)
    rho, sigma = O.smooth_knn(dist)
    w = O.membership(dist, rho, sigma)
    assert np.all(w > 0) and np.all(w <= 1)
    assert np.allclose(w.astype(np.float64).sum(1), math.log2(15), atol=3e-5)


# ----------------------------------------------------------- union (R7)
def test_conorm_examples(O):
    for a, b, expect in golden("spec_examples.json")["conorm"]:
        idx = np.array([[1], [0]], np.int32)
        w = np.array([[a], [b]], np.float32)
        indptr, col, val = O.fuzzy_union(idx, w)
        assert np.allclose(val, [expect, expect], atol=1e-7)


def test_union_matches_scipy_and_is_symmetric(O):
    import scipy.sparse as sp
    X = synth.lowrank(600, 24, seed=6)
    k = 15
    idx, dist = O.knn(X, X, k, self_offset=0)
    rho, sigma = O.smooth_knn(dist)
    w = O.membership(dist, rho, sigma)
    indptr, col, val = O.fuzzy_union(idx, w)
    n = X.shape[0]
    A = sp.csr_matrix((w.ravel().astype(np.float64), idx.ravel(), np.arange(0, n * k + 1, k)), shape=(n, n))
    B = (A + A.T - A.multiply(A.T)).tocsr()
    B.eliminate_zeros()
    B.sort_indices()
    assert np.array_equal(indptr, B.indptr)
    assert np.array_equal(col, B.indices)
    assert np.allclose(val, B.data, rtol=2 ** -23, atol=0)
    M = sp.csr_matrix((val, col, indptr), shape=(n, n))
    assert (M - M.T).count_nonzero() == 0  # bit-exact symmetry
    # sorted by (row, col)
    for i in range(n):
        assert np.all(np.diff(col[indptr[i]:indptr[i + 1]]) > 0)


# ----------------------------------------------------------- a, b (R8)
def test_fit_ab_published_defaults(O):
    for c in golden("fit_ab.json")["cases"]:
        a, b = O.fit_ab(c["min_dist"], c["spread"])
        assert abs(a - c["a"]) < c["tol"] and abs(b - c["b"]) < c["tol"]


# ----------------------------------------------------------- gradients (R12)
A_, B_ = 1.5769434603, 0.8950608779


def _fd(f, y, h=1e-6):
    g = np.zeros_like(y)
    for c in range(len(y)):
        e = np.zeros_like(y)
        e[c] = h
        g[c] = (f(y + e) - f(y - e)) / (2 * h)
    return g


@pytest.mark.parametrize("s_target", [0.05, 0.7, 3.0, 40.0])
def test_attractive_is_negative_gradient_of_minus_log_phi(O, s_target):
    yt = np.array([0.3, -1.2])
    d = np.array([1.0, 0.5]) / np.sqrt(1.25) * np.sqrt(s_target)
    yh = yt + d
    loss = lambda y: -np.log(1.0 / (1.0 + A_ * (((y - yt) ** 2).sum()) ** B_))  # -log Phi
    grad = _fd(loss, yh)
    s = float(((yh - yt) ** 2).sum())
    update = O.attr_coef(s, A_, B_) * (yh - yt)
    assert np.allclose(update, -grad, rtol=1e-5)


@pytest.mark.parametrize("s_target", [1.0, 4.0, 50.0])
def test_repulsive_is_negative_gradient_of_minus_log_one_minus_phi(O, s_target):
    yv = np.array([2.0, 1.0])
    d = np.array([0.6, -0.8]) * np.sqrt(s_target)
    yh = yv + d
    loss = lambda y: -np.log(1.0 - 1.0 / (1.0 + A_ * (((y - yv) ** 2).sum()) ** B_))  # -log(1-Phi)
    grad = _fd(loss, yh)
    s = float(((yh - yv) ** 2).sum())
    update = O.rep_coef(s, A_, B_) * (yh - yv)
    # the 0.001 stabiliser in the denominator: relative deviation 0.001/s
    assert np.allclose(update * (0.001 + s) / s, -grad, rtol=1e-5)


# ----------------------------------------------------------- schedule (R9, R10)
@pytest.mark.parametrize("r", [1.0, 0.5, 0.37, 0.1234, 0.0051, 1e-4])
def test_schedule_counts_match_closed_form(O, r):
    N = 200
    r32 = float(np.float32(r))
    due = [O.edge_due(r32, e) for e in range(1, N)]
    # number of samples through epoch E equals floor(E r): n_epochs*w/w_max samples per fit
    cum = np.cumsum(due)
    for E in (1, 7, 50, 199):
        assert cum[E - 1] == math.floor(np.float32(E) * np.float32(r32))
    if r >= 1.0:
        assert all(due)
    if r < 1.0 / N:
        assert not any(due)


def _two_vertex_graph(w=1.0):
    return np.array([0, 1, 2], np.int64), np.array([1, 0], np.int32), np.array([w, w], np.float32)


def test_sgd_attraction_conserves_center_and_contracts(O):
    X = synth.lowrank(200, 10, seed=9)
    _, _, _, _, _, (indptr, col, w) = O.fuzzy_graph(X, 10)
    Y0 = O.random_init(200, 2, seed=3)
    Y1 = O.optimize(indptr, col, w, Y0, A_, B_, n_epochs=50, e_begin=1, e_end=2, m=0, seed=1)
    # m = 0: each edge adds +g to the head and -g to the tail: centre of mass fixed
    assert np.allclose(Y1.astype(np.float64).sum(0), Y0.astype(np.float64).sum(0), atol=1e-3)

    def loss(Y):
        d2 = ((Y[np.repeat(np.arange(200), np.diff(indptr))] - Y[col]) ** 2).sum(1).astype(np.float64)
        return float((-np.log(1.0 / (1.0 + A_ * d2 ** B_)) * w).sum())
    assert loss(Y1) < loss(Y0)


def test_sgd_update_bounded_by_clip(O):
    X = synth.lowrank(150, 8, seed=2)
    _, _, _, _, _, (indptr, col, w) = O.fuzzy_graph(X, 15)
    Y0 = O.random_init(150, 2, seed=5) * np.float32(0.01)  # crowded -> large repulsion
    N = 10
    Y1 = O.optimize(indptr, col, w, Y0, A_, B_, n_epochs=N, e_begin=1, e_end=2, m=0, seed=1)
    alpha = 1 - 1 / N
    deg = np.diff(indptr)
    # each due edge moves a vertex by <= 4 alpha per component (x2: as head and as tail)
    assert np.all(np.abs(Y1 - Y0).max(1) <= 2 * 4 * alpha * deg + 1e-5)


def test_sgd_negative_sampling_repels_close_pair(O):
    indptr, col, w = _two_vertex_graph()
    for mode in ("deterministic", "hogwild"):
        Y0 = np.array([[0.0, 0.0], [0.01, 0.0]], np.float32)
        Y1 = O.optimize(indptr, col, w, Y0, A_, B_, n_epochs=10, e_begin=1, e_end=2, m=5, seed=4, mode=mode)
        assert np.linalg.norm(Y1[0] - Y1[1]) > np.linalg.norm(Y0[0] - Y0[1])
        Y0 = np.array([[0.0, 0.0], [10.0, 0.0]], np.float32)
        Y1 = O.optimize(indptr, col, w, Y0, A_, B_, n_epochs=10, e_begin=1, e_end=2, m=0, seed=4, mode=mode)
        assert np.linalg.norm(Y1[0] - Y1[1]) < np.linalg.norm(Y0[0] - Y0[1])


def test_sgd_deterministic_is_epoch_batched(O):
    # P:148 "applying the updates at the end of each epoch": the result of one epoch
    # cannot depend on the order in which vertices are stored.  Relabel vertices by a
    # permutation; the deterministic update must commute with it (the RNG counter is
    # keyed by vertex ids, so use m = 0).
    X = synth.lowrank(120, 6, seed=11)
    _, _, _, _, _, (indptr, col, w) = O.fuzzy_graph(X, 8)
    n = 120
    Y0 = O.random_init(n, 2, seed=2)
    Y1 = O.optimize(indptr, col, w, Y0, A_, B_, n_epochs=20, e_begin=3, e_end=4, m=0, mode="deterministic")
    perm = np.random.default_rng(0).permutation(n)
    inv = np.argsort(perm)
    import scipy.sparse as sp
    M = sp.csr_matrix((w, col, indptr), shape=(n, n))
    Mp = M[perm][:, perm].tocsr()
    Mp.sort_indices()
    Y1p = O.optimize(Mp.indptr.astype(np.int64), Mp.indices.astype(np.int32), Mp.data.astype(np.float32),
                     Y0[perm], A_, B_, n_epochs=20, e_begin=3, e_end=4, m=0, mode="deterministic")
    assert np.allclose(Y1p[inv], Y1, atol=1e-5)


# ----------------------------------------------------------- transform (R15)
def test_transform_zero_epochs_is_weighted_mean(O):
    Xtr = synth.lowrank(300, 12, seed=1)
    Ytr = O.random_init(300, 2, seed=1)
    Xq = synth.lowrank(340, 12, seed=1)[300:]
    idx, dist = O.knn(Xq, Xtr, 15)
    rho, sigma = O.smooth_knn(dist)
    w = O.membership(dist, rho, sigma)
    Yq = O.transform_init(idx, w, Ytr)
    ref = (w[:, :, None].astype(np.float64) * Ytr[idx]).sum(1) / w.astype(np.float64).sum(1)[:, None]
    assert np.allclose(Yq, ref, rtol=1e-6, atol=1e-6)
    Yq1 = O.transform_optimize(idx, w, Ytr, Yq, A_, B_, n_epochs_t=1)
    assert np.array_equal(Yq1, Yq)


def test_transform_row_independence(O):
    X = synth.lowrank(400, 10, seed=3)
    Xtr, Xq = X[:300], X[300:]
    Ytr = O.random_init(300, 2, seed=1)
    Y_all = O.transform(Xtr, Ytr, Xq, k=10, n_epochs=30, a=A_, b=B_, seed=5)
    Y_a = O.transform(Xtr, Ytr, Xq[:37], k=10, n_epochs=30, a=A_, b=B_, seed=5, q_offset=0)
    Y_b = O.transform(Xtr, Ytr, Xq[37:], k=10, n_epochs=30, a=A_, b=B_, seed=5, q_offset=37)
    assert np.array_equal(np.concatenate([Y_a, Y_b]), Y_all)


# ----------------------------------------------------------- trust (R16)
def _tie_free_rows(Z):
    D = ((Z[:, None, :].astype(np.float64) - Z[None, :, :]) ** 2).sum(-1)
    assert D.max() < 2 ** 24  # integer coordinates: fp32 distances are exact
    return all(len(np.unique(np.delete(D[i], i))) == Z.shape[0] - 1 for i in range(Z.shape[0]))


def _tie_free_pair(n):
    # integer data with exact fp32 distances and no distance ties within any row,
    # so fp32 and fp64 rankings coincide and sklearn's argsort is unambiguous
    for seed in range(200):
        g = np.random.default_rng(seed)
        X = g.integers(0, 1800, (n, 5))
        Y = np.clip(np.round(X[:, :2] * 1.6 + g.standard_normal((n, 2)) * 400), 0, 2895)
        if _tie_free_rows(X) and _tie_free_rows(Y):
            return X.astype(np.float32), Y.astype(np.float32)
    raise AssertionError("no tie-free seed")


def test_trust_matches_sklearn(O):
    from sklearn.manifold import trustworthiness
    X, Y = _tie_free_pair(150)
    for k in (1, 5, 15, 40):
        t = O.trustworthiness(X, Y, k)
        ref = trustworthiness(X.astype(np.float64), Y.astype(np.float64), n_neighbors=k)
        assert abs(t - ref) < 1e-12
        assert 0.5 < t < 1.0


def test_trust_identity_is_one(O):
    X = synth.lowrank(200, 5, seed=1)
    assert O.trustworthiness(X, X, 10) == 1.0


def test_trust_batching_invariance(O):
    X = synth.lowrank(150, 9, seed=2)
    Y = synth.uniform_embedding(150, 2, seed=3)
    S, pen = O.trust_penalty(X, Y, 7)
    S1, p1 = O.trust_penalty(X, Y, 7, 0, 61)
    S2, p2 = O.trust_penalty(X, Y, 7, 61, 150)
    assert S == S1 + S2 and np.array_equal(pen, np.concatenate([p1, p2]))


# ----------------------------------------------------------- end to end
def test_oracle_fit_digits_shape_quality(O):
    # S:726 acceptance analogue: digits-shaped data keeps trust >= 0.95
    X = synth.lowrank(1000, 64, blobs=10, seed=0)
    Y = O.fit(X, k=15, n_epochs=100, a=A_, b=B_, seed=1, mode="deterministic")
    assert np.all(np.isfinite(Y))
    assert O.trustworthiness(X, Y, 15) > 0.95


# ------------------------------------------------------------------- supervised adjustment (f4)
def test_supervised_adjust_spec_examples():
    """same labels unchanged; 0 vs 1 with far_dist = 5 -> x e^-5 (0.006738);
    a -1 label with unknown_dist = 1 -> x e^-1."""
    from oracle import oracle as O
    indptr = np.array([0, 2, 4, 6], np.int64)
    col = np.array([1, 2, 0, 2, 0, 1], np.int32)
    w = np.array([0.5, 0.8, 0.5, 0.25, 0.8, 0.25], np.float32)
    p, c, v = O.supervised_adjust(indptr, col, w, [0, 0, 1], far_dist=5.0, unknown_dist=1.0)
    assert np.array_equal(p, indptr) and np.array_equal(c, col)
    assert v[0] == w[0] and v[2] == w[2]                       # (0,1), (1,0): same label
    assert abs(v[1] / w[1] - 0.006737947) < 1e-6               # (0,2): 0 vs 1
    p, c, v = O.supervised_adjust(indptr, col, w, [0, -1, 0], far_dist=5.0, unknown_dist=1.0)
    assert abs(v[0] / w[0] - math.exp(-1)) < 1e-6 and v[1] == w[1]


def test_supervised_adjust_properties():
    """Symmetry preserved (the rule is symmetric in (i, j)); all-equal labels are the identity;
    tiny products are dropped below 1e-8."""
    from oracle import oracle as O
    X = synth.lowrank(300, 8, blobs=3, seed=5)
    _, _, _, _, _, (indptr, col, w) = O.fuzzy_graph(X, 10)
    p, c, v = O.supervised_adjust(indptr, col, w, np.zeros(300, np.int64))
    assert np.array_equal(p, indptr) and np.array_equal(c, col) and np.array_equal(v, w)
    lab = np.random.default_rng(0).integers(-1, 3, 300)
    p, c, v = O.supervised_adjust(indptr, col, w, lab, far_dist=5.0)
    import scipy.sparse as sp
    B = sp.csr_matrix((v, c, p), shape=(300, 300))
    assert abs(B - B.T).max() == 0
    p, c, v = O.supervised_adjust(indptr, col, w, np.arange(300), far_dist=40.0)
    assert v.size < w.size and (v >= 1e-8).all()


# ------------------------------------------------------------------- spectral init (f3, R18)
def _csr(n, edges):
    import scipy.sparse as sp
    r = [a for a, b, _ in edges] + [b for a, b, _ in edges]
    c = [b for a, b, _ in edges] + [a for a, b, _ in edges]
    v = [x for _, _, x in edges] * 2
    B = sp.csr_matrix((np.array(v, np.float32), (r, c)), shape=(n, n))
    B.sort_indices()
    return B.indptr.astype(np.int64), B.indices.astype(np.int32), B.data.astype(np.float32), B


def test_philox_vec_matches_c_oracle():
    from oracle import oracle as O
    rng = np.random.default_rng(0)
    ctr = rng.integers(0, 2**32, (50, 4), dtype=np.uint64)
    seed = int(rng.integers(0, 2**63))
    v = O.philox_vec(ctr[:, 0], ctr[:, 1], ctr[:, 2], ctr[:, 3], seed)
    for i in range(50):
        ref = O.philox4x32_10(ctr[i].astype(np.uint32), np.array([seed & 0xFFFFFFFF, seed >> 32], np.uint32))
        assert [int(x[i]) for x in v] == [int(x) for x in ref]


def test_spectral_init_spec_examples():
    """two disconnected 3-cliques -> the first non-trivial coordinate separates them
    by sign; 3-node path with unit weights -> non-trivial eigenvector prop. to (-1, 0, 1)."""
    from oracle import oracle as O
    edges = [(0, 1, 1.0), (0, 2, 1.0), (1, 2, 1.0), (3, 4, 1.0), (3, 5, 1.0), (4, 5, 1.0)]
    ip, c, w, _ = _csr(6, edges)
    Y, V = O.spectral_init(ip, c, w, 1, seed=3, iters=200)
    assert np.sign(V[0, 0]) == np.sign(V[1, 0]) == np.sign(V[2, 0]) != np.sign(V[3, 0])
    assert np.sign(V[3, 0]) == np.sign(V[4, 0]) == np.sign(V[5, 0])
    ip, c, w, _ = _csr(3, [(0, 1, 1.0), (1, 2, 1.0)])
    Y, V = O.spectral_init(ip, c, w, 1, seed=1, iters=200)
    assert abs(V[1, 0]) < 1e-8 and abs(V[0, 0] + V[2, 0]) < 1e-8
    assert np.abs(np.abs(Y[:, 0]) - np.array([10, 0, 10])).max() < 2e-3  # rescaled to [-10, 10] + noise


def test_spectral_init_matches_dense_eigensolver():
    """Three weakly linked clusters: after the iterations the 2-D subspace equals the dense
    eigensolver's (eigenvalues 2 and 3 of L = I - D^-1/2 B D^-1/2), V is orthogonal to the
    trivial vector D^1/2 1, and each column satisfies the residual bound |L v - l v| <= 1e-3 |v|."""
    from oracle import oracle as O
    rng = np.random.default_rng(2)
    edges = []
    for g in range(3):
        base = 20 * g
        for i in range(20):
            for j in range(i + 1, 20):
                if rng.random() < 0.5:
                    edges.append((base + i, base + j, float(rng.uniform(0.3, 1.0))))
    edges += [(0, 20, 0.01), (20, 40, 0.01), (40, 1, 0.01)]
    ip, c, w, B = _csr(60, edges)
    Y, V = O.spectral_init(ip, c, w, 2, seed=7, iters=500)
    deg = np.asarray(B.astype(np.float64).sum(1)).ravel()
    Dm = np.diag(1 / np.sqrt(deg))
    L = np.eye(60) - Dm @ B.toarray().astype(np.float64) @ Dm
    lam, U = np.linalg.eigh(L)
    Q = U[:, 1:3]
    s = np.linalg.svd(Q.T @ V, compute_uv=False)  # cosines of the principal angles
    assert s.min() > 1 - 1e-8
    v0 = np.sqrt(deg) / np.linalg.norm(np.sqrt(deg))
    assert np.abs(v0 @ V).max() < 1e-10
    for j in range(2):
        v = V[:, j]
        lj = v @ L @ v / (v @ v)
        assert np.linalg.norm(L @ v - lj * v) <= 1e-3 * np.linalg.norm(v)


def test_row_parallel_loops_are_thread_invariant(O):
    """The OpenMP row loops (kNN, rho/sigma, membership, transform, trust) give bit-identical
    results at 1 and at all threads: each row is one thread's sequential computation and the
    only cross-row sum is an integer one."""
    X = synth.lowrank(700, 24, blobs=5, seed=12)
    Xq = synth.lowrank(300, 24, blobs=5, seed=13)
    Y = synth.lowrank(700, 2, blobs=5, seed=14)
    A_, B_ = 1.5769434603, 0.8950608779
    out = []
    n_all = O.get_threads()
    for th in (1, max(2, n_all)):
        O.set_threads(th)
        try:
            idx, dist = O.knn(X, X, 15, self_offset=0)
            rho, sigma = O.smooth_knn(dist)
            w = O.membership(dist, rho, sigma)
            S = O.trust_penalty(X, Y, 7)
            qi, qd = O.knn(Xq, X, 15)
            qr, qs = O.smooth_knn(qd)
            qw = O.membership(qd, qr, qs)
            Yq = O.transform_init(qi, qw, Y)
            Yq = O.transform_optimize(qi, qw, Y, Yq, A_, B_, 30, m=5, seed=3)
            out.append((idx, dist, rho, sigma, w, S, Yq))
        finally:
            O.set_threads(n_all)
    def same(a, b):
        if isinstance(a, (tuple, list)):
            return len(a) == len(b) and all(same(x, y) for x, y in zip(a, b))
        return np.array_equal(np.asarray(a), np.asarray(b))
    for a, b in zip(*out):
        assert same(a, b)

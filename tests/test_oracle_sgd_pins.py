"""Pins of the oracle's SGD details that round 1 left unpinned:

* the learning-rate decay alpha_e = alpha0 (1 - e/N) (R10; alpha at e = N-1
  is alpha0/N), for the fit and for the transform;
* head-only repulsion (negative samples move the source only);
* transform negatives drawn from the training rows [0, n_train) (R15).

Each expectation is computed independently of the oracle's arithmetic: gradients by
finite differences of the objective (-log Phi), negative-sample ids from the
Random123 Philox function (pinned by its known-answer vectors in test_oracle.py) and
the multiply-shift definition v = (u n) >> 32 (R11).  A lag-by-one alpha, no decay, a
repulsion that also pushes the sampled vertex, or negatives drawn from another range
each fail one of these.
"""
import numpy as np
import pytest

A_, B_ = 1.5769434603, 0.8950608779


def _neg_log_phi(s):
    # attractive objective term -log Phi(s), Phi = 1/(1 + a s^b), s = |y_h - y_t|^2
    return np.log1p(A_ * s ** B_)


def _attr_step(yh, yt, alpha, h=1e-6):
    """-alpha * d/dyh [-log Phi(|yh - yt|^2)] by central differences (fp64)."""
    yh = np.asarray(yh, np.float64)
    yt = np.asarray(yt, np.float64)
    g = np.zeros_like(yh)
    for c in range(yh.shape[0]):
        e = np.zeros_like(yh)
        e[c] = h
        g[c] = (_neg_log_phi(((yh + e - yt) ** 2).sum()) - _neg_log_phi(((yh - e - yt) ** 2).sum())) / (2 * h)
    return -alpha * g


def _two_vertex():
    return np.array([0, 1, 2], np.int64), np.array([1, 0], np.int32), np.array([1.0, 1.0], np.float32)


@pytest.mark.parametrize("N", [10, 200])
@pytest.mark.parametrize("which", ["first", "middle", "last"])
def test_fit_alpha_decay_deterministic(O, N, which):
    indptr, col, w = _two_vertex()
    e = {"first": 1, "middle": N // 2, "last": N - 1}[which]
    alpha = 1.0 - e / N                       # R10: alpha0 = 1
    if which == "last":
        assert alpha == pytest.approx(1.0 / N)
    Y0 = np.array([[0.0, 0.0], [0.8, 0.6]], np.float32)  # s = 1: no clipping (|g| < 4)
    Y1 = O.optimize(indptr, col, w, Y0, A_, B_, n_epochs=N, e_begin=e, e_end=e + 1, m=0, seed=0,
                    mode="deterministic")
    # deterministic: both directed edges read Y_e; vertex 0 is head of (0,1) and tail of (1,0)
    g0 = _attr_step(Y0[0], Y0[1], alpha)
    g1 = _attr_step(Y0[1], Y0[0], alpha)
    np.testing.assert_allclose(Y1[0].astype(np.float64) - Y0[0], g0 - g1, rtol=2e-5, atol=2e-7)
    np.testing.assert_allclose(Y1[1].astype(np.float64) - Y0[1], g1 - g0, rtol=2e-5, atol=2e-7)


def test_fit_alpha_decay_hogwild_sequential(O):
    indptr, col, w = _two_vertex()
    N, e = 50, 49
    alpha = 1.0 / N
    Y0 = np.array([[0.0, 0.0], [0.8, 0.6]], np.float32)
    Y1 = O.optimize(indptr, col, w, Y0, A_, B_, n_epochs=N, e_begin=e, e_end=e + 1, m=0, seed=0, mode="hogwild")
    # in place, CSR order: edge (0,1) moves 0 by +g and 1 by -g, then edge (1,0) on the new positions
    y = Y0.astype(np.float64)
    g = _attr_step(y[0], y[1], alpha)
    y0 = np.float32(y[0] + g).astype(np.float64)
    y1 = np.float32(y[1] - g).astype(np.float64)
    g2 = _attr_step(y1, y0, alpha)
    np.testing.assert_allclose(Y1[1], y1 + g2, rtol=2e-5, atol=2e-7)
    np.testing.assert_allclose(Y1[0], y0 - g2, rtol=2e-5, atol=2e-7)


def _philox_word(O, seed, c, word):
    out = O.philox4x32_10([c[0], c[1], c[2], c[3]], [seed & 0xFFFFFFFF, seed >> 32])
    return int(out[word])


def _negatives(O, seed, h, t, e, m, n):
    # R11: u = Philox(key = seed, ctr = (h, t, e, p >> 2))[p & 3], v = (u n) >> 32
    return [(_philox_word(O, seed, (h, t, e, p >> 2), p & 3) * n) >> 32 for p in range(m)]


@pytest.mark.parametrize("mode", ["deterministic", "hogwild"])
def test_fit_repulsion_moves_head_only(O, mode):
    # vertices 0 <-> 1 joined, vertex 2 isolated (no edges): it can only ever be a negative
    # sample.  Head-only repulsion leaves it bit-unchanged while it still repels.
    indptr = np.array([0, 1, 2, 2], np.int64)
    col = np.array([1, 0], np.int32)
    w = np.array([1.0, 1.0], np.float32)
    N, m, seed = 20, 5, 11
    sampled = set()
    for e in range(1, N):
        for h, t in ((0, 1), (1, 0)):
            sampled.update(_negatives(O, seed, h, t, e, m, 3))
    assert 2 in sampled  # vertex 2 is drawn as a negative
    Y0 = np.array([[0.0, 0.0], [0.5, 0.0], [0.2, 0.1]], np.float32)
    Y1 = O.optimize(indptr, col, w, Y0, A_, B_, n_epochs=N, m=m, seed=seed, mode=mode)
    assert np.array_equal(Y1[2], Y0[2])
    # ... and it did act on the heads: moving it far away changes their trajectory
    Yfar = Y0.copy()
    Yfar[2] = [500.0, 500.0]
    Y2 = O.optimize(indptr, col, w, Yfar, A_, B_, n_epochs=N, m=m, seed=seed, mode=mode)
    assert not np.array_equal(Y1[:2], Y2[:2])


def test_fit_repulsion_single_negative_closed_form(O):
    # one epoch, m = 1, three vertices where the one negative of each edge is known from the
    # Philox definition: vertex h's deterministic update is 2 g_att + g_rep (or 2 g_att if the
    # sample is h itself), the repulsive step being -alpha d/dyh[-log(1 - Phi)],
    # each component clipped to 4 (none is here)
    indptr = np.array([0, 1, 2, 2], np.int64)
    col = np.array([1, 0], np.int32)
    w = np.array([1.0, 1.0], np.float32)
    N, e, seed = 4, 2, 5
    alpha = 1.0 - e / N
    Y0 = np.array([[0.0, 0.0], [1.2, 0.5], [-0.7, 1.9]], np.float32)
    Y1 = O.optimize(indptr, col, w, Y0, A_, B_, n_epochs=N, e_begin=e, e_end=e + 1, m=1, seed=seed,
                    mode="deterministic")

    def rep_step(yh, yv, h=1e-6):
        def f(y):
            s = ((y - yv) ** 2).sum()
            return -np.log(1.0 - 1.0 / (1.0 + A_ * s ** B_))
        g = np.zeros(2)
        for c in range(2):
            d = np.zeros(2)
            d[c] = h
            g[c] = (f(yh + d) - f(yh - d)) / (2 * h)
        return -alpha * g

    y = Y0.astype(np.float64)
    for h, t in ((0, 1), (1, 0)):
        v = _negatives(O, seed, h, t, e, 1, 3)[0]
        upd = _attr_step(y[h], y[t], alpha) - _attr_step(y[t], y[h], alpha)
        if v != h:
            # the oracle's repulsive coefficient carries umap-learn's 0.001 stabiliser (R12):
            # relative deviation 0.001/s from the exact gradient, s >= 1 here
            s = ((y[h] - y[v]) ** 2).sum()
            assert s >= 1.0
            upd = upd + rep_step(y[h], y[v])
            tol = 0.0011 / s * np.abs(rep_step(y[h], y[v])).max() + 1e-6
        else:
            tol = 1e-6
        np.testing.assert_allclose(Y1[h].astype(np.float64) - y[h], upd, atol=tol)
    assert np.array_equal(Y1[2], Y0[2])


def test_transform_alpha_decay_last_epoch(O):
    # one query row with one neighbour (training row 0), m = 0, only epoch N_t - 1:
    # the query moves by alpha0/N_t times the attractive step; training rows are frozen
    Ytr = np.array([[0.8, 0.6], [5.0, 5.0]], np.float32)
    Yq = np.array([[0.0, 0.0]], np.float32)
    idx = np.array([[0]], np.int32)
    w = np.array([[1.0]], np.float32)
    for Nt in (3, 67):
        Y1 = O.transform_optimize(idx, w, Ytr, Yq, A_, B_, n_epochs_t=Nt, m=0, e_begin=Nt - 1, e_end=Nt)
        np.testing.assert_allclose(Y1[0].astype(np.float64) - Yq[0], _attr_step(Yq[0], Ytr[0], 1.0 / Nt),
                                   rtol=2e-5, atol=2e-7)


def test_transform_negatives_over_training_rows(O):
    # R15 / S:530: negatives v = (u n_train) >> 32 index the training rows, none skipped
    # (the query is not a training row).  A training row influences the query iff it is
    # sampled (the neighbour t is chosen so that it is never sampled): perturbing every
    # sampled row changes the result, perturbing any other row does not.
    rng = np.random.default_rng(3)
    ntr, Nt, m, seed = 40, 4, 5, 9
    t = ntr - 1
    Ytr = rng.uniform(-3, 3, (ntr, 2)).astype(np.float32)
    Yq = np.array([[0.1, -0.2]], np.float32)
    idx = np.array([[t]], np.int32)
    w = np.array([[1.0]], np.float32)
    for q_offset in range(1000, 2000):  # a query id whose samples include row 0 but not t
        sampled = set()
        for e in range(1, Nt):
            sampled.update(_negatives(O, seed, q_offset, t, e, m, ntr))
        if 0 in sampled and t not in sampled:
            break
    assert 0 in sampled and t not in sampled and len(sampled) < ntr - 1
    base = O.transform_optimize(idx, w, Ytr, Yq, A_, B_, n_epochs_t=Nt, m=m, seed=seed, q_offset=q_offset)
    for j in range(ntr - 1):
        Yp = Ytr.copy()
        Yp[j] += np.float32(0.37)
        out = O.transform_optimize(idx, w, Yp, Yq, A_, B_, n_epochs_t=Nt, m=m, seed=seed, q_offset=q_offset)
        assert (not np.array_equal(out, base)) == (j in sampled), j

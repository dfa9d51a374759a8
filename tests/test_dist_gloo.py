"""world_size-2 gloo tests of the multi-GPU orchestration (paper_2008_00325_b200/dist.py)
on CPU.  The compute steps are injected from the oracle so the host logic (shard
ranges, global ids and offsets, the all-gather, the merge order, the all-reduce,
the partition gather) is checked against a single-process run."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


# ---- oracle-backed compute callbacks (CPU tensors in, CPU tensors out)
def _o():
    from oracle import oracle
    return oracle


def knn_cpu(Xq, Xr, k, exclude_self=False, query_offset=0, index_offset=0, squared=False):
    O = _o()
    xq, xr = Xq.numpy(), Xr.numpy()
    nq = xq.shape[0]
    idx = np.empty((nq, k), np.int32)
    d = np.empty((nq, k), np.float32)
    for i in range(nq):  # global-id self exclusion via the oracle's per-row self_offset
        own = query_offset + i - index_offset
        so = own if (exclude_self and 0 <= own < xr.shape[0]) else -1
        ri, rd = O.knn(xq[i:i + 1], xr, k, self_offset=so)
        idx[i], d[i] = ri[0] + index_offset, rd[0] ** 2 if squared else rd[0]
    return torch.from_numpy(idx), torch.from_numpy(d)


def merge_cpu(idx_parts, d2_parts, k):
    ip, dp = idx_parts.numpy(), d2_parts.numpy()
    P, n, kin = ip.shape
    out_i = np.empty((n, k), np.int32)
    out_d = np.empty((n, k), np.float32)
    for i in range(n):
        ids = ip[:, i, :].ravel()
        ds = dp[:, i, :].ravel()
        order = np.lexsort((ids, ds))[:k]
        out_i[i], out_d[i] = ids[order], np.sqrt(ds[order])
    return torch.from_numpy(out_i), torch.from_numpy(out_d)


def penalty_cpu(X, emb_idx, k, lo, hi):
    O = _o()
    x = X.numpy()
    n = x.shape[0]
    S = 0
    pen = np.zeros(hi - lo, np.int64)
    for r, i in enumerate(range(lo, hi)):
        dx = np.array([O.sqdist(x[i], x[l]) for l in range(n)], np.float32)
        for j in emb_idx[r].numpy():
            rank = 1 + sum(1 for l in range(n) if l != i and (dx[l] < dx[j] or (dx[l] == dx[j] and l < j)))
            pen[r] += max(0, rank - k)
    S = int(pen.sum())
    return S, torch.from_numpy(pen)


def transform_cpu(X_train, Y_train, Xq, q_offset=0, **kw):
    O = _o()
    return torch.from_numpy(O.transform(X_train.numpy(), Y_train.numpy(), Xq.numpy(), k=10, n_epochs=30,
                                        a=1.5769434603, b=0.8950608779, seed=5, q_offset=q_offset))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2008_00325_b200 import dist as D
        X = torch.from_numpy(synth.lowrank(130, 6, blobs=3, seed=1))
        idx, dd = D.sharded_knn(X, 7, knn_fn=knn_cpu, merge_fn=merge_cpu)
        # sharded_fit as bench.py calls it at N > 1 (the fit keyword arguments pass through;
        # the graph's k comes from the merged kNN)
        seen = {}

        def fit_knn_rec(i, d, **kw):
            seen.update(kw, k=i.shape[1])
            return i, d
        fi, fd = D.sharded_fit(X, knn_fn=knn_cpu, merge_fn=merge_cpu, fit_knn_fn=fit_knn_rec, n_neighbors=7,
                               n_epochs=5, seed=0, knn_mode="exact", sgd_mode="deterministic")
        assert seen["k"] == 7 and "n_neighbors" not in seen and seen["n_epochs"] == 5
        assert torch.equal(fi, idx) and torch.equal(fd, dd)
        Y = torch.from_numpy(synth.uniform_embedding(130, 2, seed=2))
        emb_idx, _ = knn_cpu(Y, Y, 5, exclude_self=True)
        S = D.sharded_trust_penalty(X, emb_idx, 5, penalty_fn=penalty_cpu)
        # distributed inference: rank 0 owns the model, broadcast, partitioned transform, gather
        Xall = synth.lowrank(260, 6, blobs=3, seed=3)
        Xtr = torch.from_numpy(Xall[:100]) if rank == 0 else torch.zeros((100, 6))
        Ytr = torch.from_numpy(synth.uniform_embedding(100, 2, seed=4)) if rank == 0 else torch.zeros((100, 2))
        D.broadcast_model(Xtr, Ytr)
        lo, hi = D.shard_range(160, rank, world)
        Yq = D.partitioned_transform(Xtr, Ytr, torch.from_numpy(Xall[100 + lo:100 + hi]), lo, 160,
                                     transform_fn=transform_cpu)
        # bench.py's C5 leg: the same inference through distributed_inference, the rank's shard in
        # two chunks with global query ids (the model is re-broadcast from rank 0)
        Xtr2 = torch.from_numpy(Xall[:100]) if rank == 0 else torch.zeros((100, 6))
        Ytr2 = torch.from_numpy(synth.uniform_embedding(100, 2, seed=4)) if rank == 0 else torch.zeros((100, 2))
        mid = (lo + hi) // 2
        chunks = [(torch.from_numpy(Xall[100 + lo:100 + mid]), lo), (torch.from_numpy(Xall[100 + mid:100 + hi]), mid)]
        Yq2 = D.distributed_inference(Xtr2, Ytr2, chunks, 160, transform_fn=transform_cpu)
        q.put((rank, idx.numpy(), dd.numpy(), S, Yq.numpy(), Yq2.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_gloo_world2_matches_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=540) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    O = _o()
    X = synth.lowrank(130, 6, blobs=3, seed=1)
    ri, rd = O.knn(X, X, 7, self_offset=0)
    Y = synth.uniform_embedding(130, 2, seed=2)
    S_ref, _ = O.trust_penalty(X, Y, 5)
    Xall = synth.lowrank(260, 6, blobs=3, seed=3)
    Ytr = synth.uniform_embedding(100, 2, seed=4)
    Yq_ref = O.transform(Xall[:100], Ytr, Xall[100:], k=10, n_epochs=30, a=1.5769434603, b=0.8950608779, seed=5)
    for rank, idx, dd, S, Yq, Yq2 in res:
        assert np.array_equal(idx, ri), rank
        assert np.array_equal(dd, rd), rank
        assert S == S_ref
        assert np.array_equal(Yq, Yq_ref)
        assert np.array_equal(Yq2, Yq_ref)


def test_shard_ranges_cover_rows():
    from paper_2008_00325_b200.dist import shard_range
    for n in (1, 7, 70000, 8000000):
        for world in (1, 2, 3, 8):
            r = [shard_range(n, i, world) for i in range(world)]
            assert r[0][0] == 0 and r[-1][1] == n
            assert all(r[i][1] == r[i + 1][0] for i in range(world - 1))
            assert max(h - l for l, h in r) - min(h - l for l, h in r) <= 1

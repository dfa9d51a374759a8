"""Multi-GPU orchestration over torch.distributed.

One process per GPU; NCCL over NVLink/NVSwitch for the plumbing.  Only the parts of
the path that shard naturally are distributed:

* kNN (a2): reference ("index") rows are sharded, every rank searches its shard for
  all queries with global ids and squared distances, the per-rank candidate lists
  are exchanged with one all-gather and merged by key (d2, id) -- bit-identical to
  the single-GPU result because the exact keys do not depend on the shard.
* trustworthiness (a10): rows are sharded; one int64 all-reduce of the penalty.
* transform (a9): the paper's distributed inference -- the trained model
  (X_train, Y_train) is broadcast, every rank embeds its contiguous partition (the
  RNG is keyed by the global query id, so the result is partition-invariant), and
  the partitions are gathered.
* graph build and fit SGD (a3-a8): replicated ("distributed training is an open
  problem") after the kNN merge.

The compute steps are injectable (knn_fn, merge_fn, ...) so the orchestration is
tested with the gloo backend on CPU; on GPUs they default to the CUDA library.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int):
    """Contiguous balanced rows [lo, hi) of rank."""
    return n * rank // world, n * (rank + 1) // world


def _rank_world(group):
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def _default_knn():
    from . import api
    return api.knn


def _default_merge():
    from . import api
    return api.topk_merge


def sharded_knn(X, k, group=None, knn_fn=None, merge_fn=None, phase_mark=None):
    """Exact kNN of every row of X against X (self excluded), reference rows sharded
    across the ranks of `group`.  Returns (idx int32 n x k, dist fp32 n x k), identical
    on every rank.  phase_mark (optional): called with "searched" and "gathered" at the
    phase boundaries (bench.py records CUDA events there)."""
    knn_fn = knn_fn or _default_knn()
    merge_fn = merge_fn or _default_merge()
    rank, world = _rank_world(group)
    n = X.shape[0]
    lo, hi = shard_range(n, rank, world)
    if hi - lo < k + 1:
        raise ValueError(f"shard of {hi - lo} rows is too small for k={k}")
    ci, cd = knn_fn(X, X[lo:hi], k, exclude_self=True, query_offset=0, index_offset=lo, squared=True)
    if phase_mark:
        phase_mark("searched")
    if world == 1:
        if phase_mark:
            phase_mark("gathered")
        return merge_fn(ci[None], cd[None], k)
    gi = [torch.empty_like(ci) for _ in range(world)]
    gd = [torch.empty_like(cd) for _ in range(world)]
    dist.all_gather(gi, ci.contiguous(), group=group)
    dist.all_gather(gd, cd.contiguous(), group=group)
    if phase_mark:
        phase_mark("gathered")
    return merge_fn(torch.stack(gi), torch.stack(gd), k)


def sharded_trust_penalty(X, emb_idx, k, group=None, penalty_fn=None, knn_mode="exact", Y=None):
    """Integer trust penalty S with rows sharded; one all-reduce.  emb_idx: n x k embedding kNN;
    Y (optional) the embedding, a layout hint for the tensor path."""
    if penalty_fn is None:
        from . import api

        def penalty_fn(X, e, k, lo, hi):
            return api.trust_penalty(X, e, k, lo, hi, knn_mode=knn_mode, Y=Y)
    rank, world = _rank_world(group)
    n = X.shape[0]
    lo, hi = shard_range(n, rank, world)
    S, _ = penalty_fn(X, emb_idx[lo:hi].contiguous(), k, lo, hi)
    if world == 1:
        return int(S)
    t = torch.tensor([S], dtype=torch.int64, device=X.device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return int(t.item())


def sharded_trustworthiness(X, Y, k, group=None, knn_fn=None, penalty_fn=None, knn_mode="exact"):
    """T(k) with the input-space rank counts sharded by rows (R16)."""
    knn_fn = knn_fn or _default_knn()
    emb_idx, _ = knn_fn(Y, Y, k, exclude_self=True)
    S = sharded_trust_penalty(X, emb_idx, k, group=group, penalty_fn=penalty_fn, knn_mode=knn_mode, Y=Y)
    from . import api
    return api.trust_from_penalty(S, X.shape[0], k), S


def sharded_fit(X, group=None, knn_fn=None, merge_fn=None, fit_knn_fn=None, **kw):
    """Fit with the kNN sharded over the group, graph + SGD replicated on every rank."""
    if fit_knn_fn is None:
        from . import api
        fit_knn_fn = api.fit_knn
    if knn_fn is None:
        from . import api
        mode = kw.get("knn_mode", "exact")

        def knn_fn(Xq, Xr, k, **a):
            return api.knn(Xq, Xr, k, mode=mode, **a)
    k = kw.pop("n_neighbors", 15)  # fit_knn takes k from the graph's shape
    idx, dst = sharded_knn(X, k, group=group, knn_fn=knn_fn, merge_fn=merge_fn)
    return fit_knn_fn(idx, dst, **kw)


def broadcast_model(X_train, Y_train, group=None, src=0):
    """Broadcast the trained model (X_train, Y_train) from `src` (the model is
    sent to every worker).  Non-src ranks pass tensors of the right shape."""
    _, world = _rank_world(group)
    if world > 1:
        dist.broadcast(X_train, src=src, group=group)
        dist.broadcast(Y_train, src=src, group=group)
    return X_train, Y_train


def partitioned_transform(X_train, Y_train, Xq_local, q_offset, n_total, group=None, transform_fn=None,
                          gather=True, **kw):
    """Embed this rank's partition (global rows [q_offset, q_offset + len)) against the
    broadcast model; optionally all-gather the partitions (every rank gets n_total rows)."""
    if transform_fn is None:
        from . import api
        transform_fn = api.transform
    Yq = transform_fn(X_train, Y_train, Xq_local, q_offset=q_offset, **kw)
    rank, world = _rank_world(group)
    if world == 1 or not gather:
        return Yq
    lo, hi = shard_range(n_total, rank, world)
    assert (lo, hi - lo) == (q_offset, Yq.shape[0]), "partition must follow shard_range"
    m = max(shard_range(n_total, r, world)[1] - shard_range(n_total, r, world)[0] for r in range(world))
    pad = torch.zeros((m, Yq.shape[1]), dtype=Yq.dtype, device=Yq.device)
    pad[:Yq.shape[0]] = Yq
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    out = [parts[r][:shard_range(n_total, r, world)[1] - shard_range(n_total, r, world)[0]] for r in range(world)]
    return torch.cat(out)


def distributed_inference(X_train, Y_train, chunks, n_total, group=None, transform_fn=None, src=0, **kw):
    """The paper's distributed UMAP inference (App. B): the model (X_train, Y_train)
    trained on rank `src` is broadcast, every rank embeds its partition -- a list of
    (Xq_chunk, q_offset) with global query ids, whose chunks together cover shard_range(n_total,
    rank, world) in order -- and the partitions are all-gathered (every rank gets n_total rows).
    Bit-identical for any world size: each query row depends only on the model and its global
    id (R15)."""
    if transform_fn is None:
        from . import api
        transform_fn = api.transform
    broadcast_model(X_train, Y_train, group=group, src=src)
    rank, world = _rank_world(group)
    lo, hi = shard_range(n_total, rank, world)
    parts = []
    nxt = lo
    for Xq, off in chunks:
        assert off == nxt, "chunks must cover the rank's shard in order"
        parts.append(transform_fn(X_train, Y_train, Xq, q_offset=off, **kw))
        nxt = off + Xq.shape[0]
    assert nxt == hi, "chunks must cover the rank's shard"
    Yq = torch.cat(parts) if len(parts) > 1 else parts[0]
    if world == 1:
        return Yq
    m = max(shard_range(n_total, r, world)[1] - shard_range(n_total, r, world)[0] for r in range(world))
    pad = torch.zeros((m, Yq.shape[1]), dtype=Yq.dtype, device=Yq.device)
    pad[:Yq.shape[0]] = Yq
    out = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(out, pad, group=group)
    return torch.cat([out[r][:shard_range(n_total, r, world)[1] - shard_range(n_total, r, world)[0]]
                      for r in range(world)])

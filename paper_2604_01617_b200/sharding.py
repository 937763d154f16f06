"""Multi-GPU execution of the hot path: one process per GPU.

* Routing shards QUERIES over replicas of the index: rank r routes its contiguous block of
  queries with their global query indices (so entry points are those of the single-GPU run,
  router.py:42-45), and the results are gathered in rank order (``search_batch_sharded`` for
  host arrays; ``search_batch_sharded_device`` keeps queries, results and the all-gather on
  the GPUs).  Output is identical to the single-GPU ``search_batch``.
* Exhaustive AUTO top-k shards the NODES: each rank keeps an exact local top-k over its node
  range (global ids), then ONE exchange step (all-gather of q x k (dist, id) lists) and a
  merge by (dist, id) give the exact global top-k of ``oracle_auto_topk``
  (evaluate.py:32-55): every member of the global top-k is in its shard's local top-k.

Collectives go through ``torch.distributed`` (NCCL on GPUs, gloo for the CPU tests).  With
no process group initialised both functions run single-process.
"""

from __future__ import annotations

import numpy as np


def comm(group=None):
    """(rank, world) of the default/global process group, or (0, 1) when not initialised."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of `total` items owned by `rank` (sizes differ by <= 1)."""
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def all_gather_rows(arr: np.ndarray, group=None) -> list[np.ndarray]:
    """All-gather a per-rank 2-D array with a variable number of rows; returns the list of
    every rank's array, in rank order."""
    import torch
    import torch.distributed as dist
    rank, world = comm(group)
    if world == 1:
        return [arr]
    device = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    arr = np.ascontiguousarray(arr)
    rows = torch.tensor([arr.shape[0]], dtype=torch.int64, device=device)
    all_rows = [torch.zeros_like(rows) for _ in range(world)]
    dist.all_gather(all_rows, rows, group=group)
    counts = [int(r.item()) for r in all_rows]
    cap = max(counts)
    width = arr.shape[1] if arr.ndim == 2 else 1
    # move raw bytes so every dtype (f64, i64) travels exactly
    raw = arr.reshape(arr.shape[0], width).view(np.uint8).reshape(arr.shape[0], -1)
    pad = np.zeros((cap, raw.shape[1]), np.uint8)
    pad[: raw.shape[0]] = raw
    t = torch.from_numpy(pad).to(device)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    res = []
    for c, o in zip(counts, out):
        b = o.cpu().numpy()[:c]
        res.append(np.ascontiguousarray(b).view(arr.dtype).reshape((c,) + arr.shape[1:]))
    return res


def search_batch_sharded(graph, query_features, query_attrs, params, masks=None, group=None,
                         route_fn=None):
    """search_batch (router.py:98-124) with the queries split across ranks.

    route_fn(qf, qa, masks, qi0) -> (ids, dists, stats) runs one shard; the default is the
    B200 path (``search_batch_arrays`` on this rank's GPU).  Returns the full (ids, dists,
    stats) on every rank."""
    from .router import search_batch_arrays
    qf = np.asarray(query_features)
    qa = np.asarray(query_attrs)
    rank, world = comm(group)
    lo, hi = shard_range(qf.shape[0], rank, world)
    mk = None if masks is None else np.asarray(masks)[lo:hi]
    if route_fn is None:
        def route_fn(f, a, m, qi0):
            return search_batch_arrays(graph, f, a, params, masks=m, qi0=qi0)
    ids, dists, stats = route_fn(qf[lo:hi], qa[lo:hi], mk, lo)
    parts = [all_gather_rows(np.asarray(x), group) for x in (ids, dists, stats)]
    return tuple(np.concatenate(p, axis=0) for p in parts)


def search_batch_sharded_device(dev, qf_d, qa_d, q: int, k: int, pioneer: int, inv_alpha: float,
                                qm_d=None, seed: int = 0, group=None, use_coarse: bool = True):
    """search_batch with the queries split across ranks, everything on the device.

    qf_d / qa_d (/ qm_d): the full q-row query batch as float64 CUDA tensors on every rank;
    ``dev`` is this rank's DeviceIndex (a replica of the index), launching on the current torch
    stream.  Rank r routes rows [r*cap, min(q, (r+1)*cap)) with cap = ceil(q / world) and their
    global query indices (so entry points are the single-GPU run's, router.py:42-45); one
    all_gather_into_tensor per output (NCCL over NVLink) assembles the results in rank order.
    Returns CUDA tensors (ids int64 q x k, dists float64 q x k, stats int64 q x 5), identical to
    the single-GPU call."""
    import torch
    import torch.distributed as dist
    rank, world = comm(group)
    cap = (q + world - 1) // world
    lo = min(q, rank * cap)
    hi = min(q, lo + cap)
    dv = qf_d.device
    ids = torch.empty((cap, k), dtype=torch.int64, device=dv)
    dists = torch.empty((cap, k), dtype=torch.float64, device=dv)
    st = torch.zeros((cap, 5), dtype=torch.int64, device=dv)
    if hi > lo:
        if dv.type == "cuda":
            dev.set_stream(torch.cuda.current_stream(dv).cuda_stream)
        dev.route_dev(qf_d[lo:hi].data_ptr(), qa_d[lo:hi].data_ptr(),
                      None if qm_d is None else qm_d[lo:hi].data_ptr(), hi - lo, k, pioneer,
                      inv_alpha, ids.data_ptr(), dists.data_ptr(), st.data_ptr(), seed=seed,
                      qi0=lo, use_coarse=use_coarse)
    if world == 1:
        return ids[:q], dists[:q], st[:q]
    out = []
    for t in (ids, dists, st):
        full = torch.empty((world * cap,) + tuple(t.shape[1:]), dtype=t.dtype, device=dv)
        dist.all_gather_into_tensor(full, t, group=group)
        out.append(full[:q])
    return tuple(out)


def merge_topk(dist_lists, id_lists, k: int):
    """Per-query exact merge of candidate lists by (dist, id); inf-padded entries sort last."""
    d = np.concatenate(dist_lists, axis=1)
    i = np.concatenate(id_lists, axis=1)
    order = np.lexsort((i, d), axis=-1)[:, :k]
    return np.take_along_axis(i, order, 1), np.take_along_axis(d, order, 1)


def oracle_auto_topk_sharded(features, attrs, query_features, query_attrs, k: int, config,
                             masks=None, group=None, local_fn=None):
    """oracle_auto_topk over all queries with the node set split across ranks.

    local_fn(features_shard, attrs_shard, qf, qa, k_local, masks) -> (ids, dists) is the
    exact local top-k of one shard (shard-local ids); the default is the B200 path
    (``oracle_auto_topk_batch`` on this rank's GPU).  Returns (ids, dists) on every rank."""
    from .evaluate import oracle_auto_topk_batch
    features = np.asarray(features)
    attrs = np.asarray(attrs)
    n = features.shape[0]
    if not 1 <= k <= n:
        raise ValueError(f"k={k} must be in [1, n={n}]")
    rank, world = comm(group)
    lo, hi = shard_range(n, rank, world)
    qf = np.atleast_2d(np.asarray(query_features, np.float64))
    qa = np.atleast_2d(np.asarray(query_attrs))
    q = qf.shape[0]
    kl = min(k, hi - lo)
    ids = np.full((q, k), np.iinfo(np.int64).max, np.int64)
    dists = np.full((q, k), np.inf, np.float64)
    if kl > 0:
        if local_fn is None:
            def local_fn(f, a, qf_, qa_, kk, m):
                return oracle_auto_topk_batch(f, a, qf_, qa_, kk, config, m, return_dists=True)
        li, ld = local_fn(features[lo:hi], attrs[lo:hi], qf, qa, kl, masks)
        ids[:, :kl] = np.asarray(li, np.int64) + lo
        dists[:, :kl] = ld
    # the exchange step: every rank's q x k candidates, then an exact (dist, id) merge
    return merge_topk(all_gather_rows(dists, group), all_gather_rows(ids, group), k)

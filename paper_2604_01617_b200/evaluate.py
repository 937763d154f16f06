"""Exact AUTO ground truth on the device, recall, and the benchmark sweep
(reference evaluate.py:32-158)."""

from __future__ import annotations

import csv
import time
from dataclasses import dataclass

import numpy as np

from .device import DeviceIndex
from .graph import RelationGraph
from .metric import MetricConfig
from .router import SearchParams, search_batch_arrays

CSV_FIELDS = ["k", "pioneer", "mean_recall_at_10", "qps", "mean_dist_evals", "n_queries"]

_CACHE: dict = {}


def _device_for(features, attrs) -> DeviceIndex:
    key = (features.__array_interface__["data"][0], features.shape,
           attrs.__array_interface__["data"][0], attrs.shape)
    d = _CACHE.get(key)
    if d is None or d.features is not features and not np.shares_memory(d.features, features):
        _CACHE.clear()
        d = DeviceIndex(features, attrs, 2)
        _CACHE[key] = d
    return d


def oracle_auto_topk_batch(features, attrs, query_features, query_attrs, k: int,
                           config: MetricConfig, masks=None, return_dists=False):
    """oracle_auto_topk for many queries in one device pass (q x k int64 ids)."""
    features = np.ascontiguousarray(features, np.float32)
    attrs = np.ascontiguousarray(attrs, np.int32)
    n = features.shape[0]
    if k > n:
        raise ValueError(f"k={k} exceeds dataset size {n}")
    if k < 1:
        raise ValueError("k must be >= 1")
    dev = _device_for(features, attrs)
    ids, dists = dev.bf_topk_queries(query_features, query_attrs, k, config.alpha, masks)
    return (ids, dists) if return_dists else ids


def oracle_auto_topk(features, attrs, query_feature, query_attrs, k: int, config: MetricConfig,
                     mask=None) -> np.ndarray:
    """Exact top-k under the fused metric by full scan, ties by ascending id."""
    qm = None if mask is None else np.asarray(mask)[None]
    return oracle_auto_topk_batch(features, attrs, np.asarray(query_feature)[None],
                                  np.asarray(query_attrs)[None], k, config, qm)[0]


def oracle_hybrid_groundtruth(features, attrs, query_feature, query_attrs, k: int, mask=None):
    """Exact-match filter then Euclidean rank (reference evaluate.py:58-77); host NumPy."""
    adiff = np.abs(np.asarray(attrs, np.int64) - np.asarray(query_attrs, np.int64))
    if mask is not None:
        adiff = adiff * np.asarray(mask, np.int64)
    matching = np.nonzero(adiff.sum(axis=1) == 0)[0]
    if matching.size == 0:
        return np.empty(0, dtype=np.int64)
    diff = np.asarray(features)[matching].astype(np.float64) - np.asarray(query_feature, np.float64)
    s_v = np.sqrt((diff * diff).sum(axis=1))
    order = np.lexsort((matching, s_v))
    return matching[order[: min(k, matching.size)]]


def recall_at_k(retrieved, ground_truth, k: int) -> float:
    """|first-k(retrieved) ∩ gt| / min(k, |gt|); empty gt -> 1.0 (reference evaluate.py:80-92)."""
    if k < 1:
        raise ValueError("k must be >= 1")
    gt = set(int(x) for x in ground_truth)
    if not gt:
        return 1.0
    top = [int(x) for x in list(retrieved)[:k]]
    return len(gt.intersection(top)) / min(k, len(gt))


def mean_recall(ids: np.ndarray, gt: np.ndarray, k: int = 10) -> float:
    """Vectorised mean recall@k for full-width ground truth rows (q x >= k, no -1)."""
    top = ids[:, :k]
    g = gt[:, :k]
    hits = (top[:, :, None] == g[:, None, :]).any(axis=2).sum(axis=1)
    return float((hits / min(k, g.shape[1])).mean())


@dataclass(frozen=True)
class SweepRow:
    k: int
    pioneer: int
    mean_recall_at_10: float
    qps: float
    mean_dist_evals: float
    n_queries: int


def bench_sweep(graph: RelationGraph, query_features, query_attrs, ground_truth, k_values,
                masks=None, seed: int = 0, pioneer_size: int | None = None,
                timing_passes: int = 3) -> list[SweepRow]:
    """K sweep with the reference's semantics (evaluate.py:95-141): mean Recall@10 from the
    first pass, QPS = q / median wall time of the passes, mean distance evaluations.  Each
    pass is one batched device call through the public search API."""
    if ground_truth is None or len(ground_truth) != query_features.shape[0]:
        raise ValueError("ground truth missing or query count mismatch")
    q = query_features.shape[0]
    rows = []
    for k in k_values:
        if k > graph.n:
            raise ValueError(f"k={k} exceeds dataset size {graph.n}")
        params = SearchParams(k=k, pioneer_size=pioneer_size, seed=seed)
        elapsed = []
        recalls = evals = None
        for p in range(max(1, timing_passes)):
            t0 = time.perf_counter()
            ids, _, st = search_batch_arrays(graph, query_features, query_attrs, params, masks)
            elapsed.append(time.perf_counter() - t0)
            if p == 0:
                recalls = np.array([recall_at_k(ids[i], ground_truth[i], 10) for i in range(q)])
                evals = st[:, 0].astype(np.float64)
        rows.append(SweepRow(k=k, pioneer=params.resolved_pioneer_size(),
                             mean_recall_at_10=float(recalls.mean()),
                             qps=q / float(np.median(elapsed)),
                             mean_dist_evals=float(evals.mean()), n_queries=q))
    return rows


def write_sweep_csv(path, rows) -> None:
    with open(path, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=CSV_FIELDS)
        w.writeheader()
        for r in rows:
            w.writerow({"k": r.k, "pioneer": r.pioneer,
                        "mean_recall_at_10": f"{r.mean_recall_at_10:.6f}",
                        "qps": f"{r.qps:.2f}", "mean_dist_evals": f"{r.mean_dist_evals:.2f}",
                        "n_queries": r.n_queries})

"""Exact AUTO ground truth on the device, recall, and the benchmark sweep
(reference evaluate.py:32-158)."""

from __future__ import annotations

import csv
import time
from dataclasses import dataclass

import numpy as np

from ._lib import fingerprint
from .device import DeviceIndex
from .graph import RelationGraph
from .metric import MetricConfig
from .router import SearchParams, search_batch_arrays

CSV_FIELDS = ["k", "pioneer", "mean_recall_at_10", "qps", "mean_dist_evals", "n_queries"]
# the reference's columns plus the routing roofline of each row: algorithmic
# bytes = dist_evals*(4d+4L) + 4*(expansions + neighbours scanned), over the median pass time
ROOFLINE_FIELDS = CSV_FIELDS + ["algorithmic_gbs", "hbm_frac"]

_CACHE: dict = {}


def clear_device_cache() -> None:
    """Drop the device copy of the last dataset passed to the oracles."""
    _CACHE.clear()


def _device_for(features, attrs) -> DeviceIndex:
    """The resident device copy of (features, attrs), re-uploaded whenever their contents
    differ from the cached copy's (a content fingerprint, not the buffer address, is the key:
    the reference oracle is a pure function of its inputs)."""
    key = (fingerprint(features), fingerprint(attrs))
    d = _CACHE.get(key)
    if d is None:
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


def oracle_hybrid_groundtruth_batch(features, attrs, query_features, query_attrs, k: int,
                                    masks=None) -> list[np.ndarray]:
    """oracle_hybrid_groundtruth for many queries in one device pass: a list of int64 id
    arrays, each of length min(k, matching nodes)."""
    features = np.ascontiguousarray(features, np.float32)
    attrs = np.ascontiguousarray(attrs, np.int32)
    dev = _device_for(features, attrs)
    ids, _, counts = dev.hybrid_groundtruth(query_features, query_attrs, int(k), masks)
    return [ids[i, : counts[i]] for i in range(ids.shape[0])]


def oracle_hybrid_groundtruth(features, attrs, query_feature, query_attrs, k: int, mask=None):
    """Nodes exactly matching the (masked) attribute constraint, ranked by pure feature
    distance, ties by id; may return fewer than k ids when matches are scarce (reference
    evaluate.py:58-77).  Runs on the device (bf_sort.cu, hybrid mode)."""
    qm = None if mask is None else np.asarray(mask)[None]
    return oracle_hybrid_groundtruth_batch(features, attrs, np.asarray(query_feature)[None],
                                           np.asarray(query_attrs)[None], k, qm)[0]


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
    # roofline columns (not in the reference's SweepRow; defaults keep its constructor)
    algorithmic_gbs: float = 0.0
    hbm_frac: float = 0.0


def routing_bytes(stats: np.ndarray, d: int, l: int) -> float:
    """SURVEY §8(d) algorithmic bytes of a routing batch from its q x 5 stats
    (dist_evals, phase1_evals, phase1_expansions, hops, scanned)."""
    st = np.asarray(stats, np.float64)
    return float(st[:, 0].sum() * (4 * d + 4 * l) + 4.0 * (st[:, 2].sum() + st[:, 3].sum() + st[:, 4].sum()))


def bench_sweep(graph: RelationGraph, query_features, query_attrs, ground_truth, k_values,
                masks=None, seed: int = 0, pioneer_size: int | None = None,
                timing_passes: int = 3, hbm_peak_gbs: float = 8000.0) -> list[SweepRow]:
    """K sweep with the reference's semantics (evaluate.py:95-141): mean Recall@10 from the
    first pass, QPS = q / median wall time of the passes, mean distance evaluations.  Each
    pass is one batched device call through the public search API.  Each row also carries
    the routing roofline: §8(d) algorithmic bytes per pass / median pass time, and its
    fraction of ``hbm_peak_gbs`` (8,000 GB/s north-star figure unless a measured peak is
    given)."""
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
                nbytes = routing_bytes(st, graph.features.shape[1], graph.attrs.shape[1])
        t = float(np.median(elapsed))
        gbs = nbytes / t / 1e9 if t > 0 else 0.0
        rows.append(SweepRow(k=k, pioneer=params.resolved_pioneer_size(),
                             mean_recall_at_10=float(recalls.mean()),
                             qps=q / t, mean_dist_evals=float(evals.mean()), n_queries=q,
                             algorithmic_gbs=gbs, hbm_frac=gbs / hbm_peak_gbs))
    return rows


def write_sweep_csv(path, rows, roofline: bool = False) -> None:
    """The reference's CSV (evaluate.py:144-158); ``roofline=True`` appends the two roofline
    columns (ROOFLINE_FIELDS)."""
    with open(path, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=ROOFLINE_FIELDS if roofline else CSV_FIELDS)
        w.writeheader()
        for r in rows:
            row = {"k": r.k, "pioneer": r.pioneer,
                   "mean_recall_at_10": f"{r.mean_recall_at_10:.6f}",
                   "qps": f"{r.qps:.2f}", "mean_dist_evals": f"{r.mean_dist_evals:.2f}",
                   "n_queries": r.n_queries}
            if roofline:
                row.update(algorithmic_gbs=f"{r.algorithmic_gbs:.1f}", hbm_frac=f"{r.hbm_frac:.4f}")
            w.writerow(row)

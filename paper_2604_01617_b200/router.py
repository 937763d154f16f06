"""Dynamic Heterogeneity Routing search API (reference router.py:19-124).

``search`` and ``search_batch`` keep the reference's signatures, validation messages and
return types; ``search_batch`` is one device call for all queries instead of a Python loop
(query_index = row number, router.py:120).  Entry points are drawn on the device with a
bit-exact port of the reference's NumPy stream (router.py:42-45).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .device import entry_points_host
from .graph import RelationGraph


@dataclass
class SearchParams:
    k: int
    pioneer_size: int | None = None  # default: max(1, k // 2)
    seed: int = 0
    mask: np.ndarray | None = None
    use_coarse: bool = True

    def resolved_pioneer_size(self) -> int:
        p = self.pioneer_size if self.pioneer_size is not None else max(1, self.k // 2)
        if not 1 <= p <= self.k:
            raise ValueError(f"pioneer_size {p} must be in [1, k={self.k}]")
        return p


@dataclass(frozen=True)
class SearchStats:
    dist_evals: int
    phase1_evals: int
    phase1_expansions: int
    hops: int


def entry_points(n: int, k: int, seed: int, query_index: int) -> np.ndarray:
    """K distinct uniform entry nodes, the reference's per-query NumPy stream."""
    return entry_points_host(n, k, seed, query_index, 1)[0]


def _validate(graph: RelationGraph, params: SearchParams):
    if not graph.frozen:
        raise ValueError("graph must be frozen before searching")
    if params.k > graph.n:
        raise ValueError(f"k={params.k} exceeds dataset size {graph.n}")
    if params.k < 1:
        raise ValueError("k must be >= 1")


def _query_arrays(graph, qf, qa):
    qf = np.ascontiguousarray(qf, dtype=np.float64)
    qa = np.ascontiguousarray(qa, dtype=np.float64)
    m, l = graph.features.shape[1], graph.attrs.shape[1]
    if qf.shape[-1] != m or (qf.ndim == 2 and qf.shape[1] != m):
        raise ValueError(f"query feature dimension {qf.shape} != {m}")
    if qa.shape[-1] != l:
        raise ValueError(f"query attribute dimension {qa.shape} != {l}")
    return qf, qa


def search(graph: RelationGraph, query_feature, query_attrs, params: SearchParams,
           query_index: int = 0):
    """Top-k ids (ascending fused distance, id tie-break) plus SearchStats."""
    _validate(graph, params)
    qf = np.ascontiguousarray(query_feature, dtype=np.float64)
    qa = np.ascontiguousarray(query_attrs, dtype=np.float64)
    if qf.shape != (graph.features.shape[1],):
        raise ValueError(f"query feature dimension {qf.shape} != {graph.features.shape[1]}")
    if qa.shape != (graph.attrs.shape[1],):
        raise ValueError(f"query attribute dimension {qa.shape} != {graph.attrs.shape[1]}")
    qm = None
    if params.mask is not None:
        qm = np.ascontiguousarray(params.mask, dtype=np.float64)
        if qm.shape != qa.shape:
            raise ValueError("mask length must equal attribute dimension")
    pioneer = params.resolved_pioneer_size()
    ids, dists, st = graph.device().route(qf[None], qa[None], params.k, pioneer,
                                          1.0 / graph.metric.alpha, qmask=None if qm is None else qm[None],
                                          seed=params.seed, qi0=query_index,
                                          use_coarse=params.use_coarse)
    s = st[0]
    return ids[0], dists[0], SearchStats(int(s[0]), int(s[1]), int(s[2]), int(s[3]))


def search_batch_arrays(graph: RelationGraph, query_features, query_attrs, params: SearchParams,
                        masks=None, qi0: int = 0):
    """search_batch returning the stats as an int64 array (q, 5): the four SearchStats
    counters plus neighbours scanned."""
    _validate(graph, params)
    qf = np.ascontiguousarray(query_features, dtype=np.float64)
    qa = np.ascontiguousarray(query_attrs, dtype=np.float64)
    q = qf.shape[0]
    if qf.ndim != 2 or qf.shape[1] != graph.features.shape[1]:
        raise ValueError(f"query feature dimension {qf.shape} != {graph.features.shape[1]}")
    if qa.shape != (q, graph.attrs.shape[1]):
        raise ValueError(f"query attribute dimension {qa.shape} != {graph.attrs.shape[1]}")
    qm = None
    if masks is not None:
        qm = np.ascontiguousarray(masks, dtype=np.float64)
        if qm.shape != qa.shape:
            raise ValueError("mask length must equal attribute dimension")
    elif params.mask is not None:
        one = np.ascontiguousarray(params.mask, dtype=np.float64)
        if one.shape != (qa.shape[1],):
            raise ValueError("mask length must equal attribute dimension")
        qm = np.broadcast_to(one, qa.shape).copy()
    pioneer = params.resolved_pioneer_size()
    return graph.device().route(qf, qa, params.k, pioneer, 1.0 / graph.metric.alpha, qmask=qm,
                                seed=params.seed, qi0=qi0, use_coarse=params.use_coarse)


def search_batch(graph: RelationGraph, query_features, query_attrs, params: SearchParams,
                 masks=None):
    """One search per query row in a single device call; query_index is the row number."""
    ids, dists, st = search_batch_arrays(graph, query_features, query_attrs, params, masks)
    stats = [SearchStats(int(r[0]), int(r[1]), int(r[2]), int(r[3])) for r in st]
    return ids, dists, stats

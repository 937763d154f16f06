"""Parity at scale and the paths added for any k / the exact-match ground truth.

* Every BASELINE config recipe (tools/configs.py) at N = 100,000 with the reference's default
  BuildParams (gamma = gamma_new = 100, sigma = 0.44): the GPU HELP graph equals the graph the
  CPU oracle builds (oracle/stable_oracle.c, parallel restatement pinned to the reference's
  loops in tests/test_oracle_golden.py) bit for bit, routing (ids, fp64 distances, all four
  SearchStats counters) and exact AUTO top-k equal the oracle's on a query sample.  cfg 3 and
  cfg 4 exercise reinforce_pass's overflow rows (_kernels.py:336-395).
* exhaustive top-k for k beyond the tiled kernels (the full-sort kernel, bf_sort.cu).
* oracle_hybrid_groundtruth on the device (evaluate.py:58-77).
* results returned through the page-locked pool stay valid across later calls.
"""

import numpy as np
import pytest

import paper_2604_01617_b200 as sb
from paper_2604_01617_b200.device import DeviceIndex
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _build_pair(cfg, n):
    from tools.configs import make_config
    X, A, QX, QA, card = make_config(cfg, n)
    m = sb.compute_alpha(sb.sample_statistics(X, A, min(1000, n), seed=0), n, A.shape[1])
    schema = sb.AttributeSchema(tuple(tuple(str(i) for i in range(c)) for c in card))
    g = sb.build(X, A, schema, sb.BuildParams(), m)
    og = O.build(X, A, m.alpha, sigma=0.44, gamma=100, gamma_new=100, nthreads=0)
    return X, A, QX, QA, m, g, og


@pytest.mark.parametrize("cfg,n,overflow", [
    ("cfg2", 100_000, False), ("cfg3", 100_000, False), ("cfg3", 20_000, True),
    ("cfg4", 100_000, True), ("cfg5c1000", 100_000, False), ("cfg5c10", 100_000, False),
    ("cfg5c1", 100_000, True)])
def test_config_recipes_at_100k(cfg, n, overflow):
    """(cfg 3 overflows at 20k, not at 100k: both are run.)"""
    X, A, QX, QA, m, g, og = _build_pair(cfg, n)
    # the descent took the same path (psi history gates the iteration count)
    assert g.build_log["psi_history"] == og.log["psi_history"]
    assert g.build_log["pairs"] == og.log["pairs"]
    np.testing.assert_array_equal(g.nbr_counts, og.nbr_counts)
    mask = np.arange(g.nbr_ids.shape[1])[None, :] < og.nbr_counts[:, None]
    np.testing.assert_array_equal(np.where(mask, g.nbr_ids, -1), np.where(mask, og.nbr_ids, -1))
    np.testing.assert_array_equal(np.where(mask, g.nbr_dists, 0), np.where(mask, og.nbr_dists, 0))
    if overflow:  # the exact sequential re-prune of full rows ran (and matched)
        assert og.log["full_merges"] > 0
        assert g.build_log["reinforce_overflow_rows"] > 0
    q = 200
    for k in (10, 100):
        got = sb.search_batch_arrays(g, QX[:q], QA[:q], sb.SearchParams(k=k))
        want = O.search_batch(X, A, og.nbr_ids, og.nbr_counts, m.alpha, QX[:q], QA[:q], k,
                              nthreads=0)
        np.testing.assert_array_equal(got[0], want[0], err_msg=f"{cfg} K={k}")
        np.testing.assert_array_equal(got[1], want[1], err_msg=f"{cfg} K={k}")
        np.testing.assert_array_equal(got[2][:, :4], want[2], err_msg=f"{cfg} K={k}")
    ti, td = sb.oracle_auto_topk_batch(X, A, QX[:40], QA[:40], 10, m, return_dists=True)
    for i in range(40):
        wi, wd = O.oracle_auto_topk(X, A, QX[i], QA[i], 10, m.alpha, return_dists=True)
        np.testing.assert_array_equal(ti[i], wi)
        np.testing.assert_array_equal(td[i], wd)


@pytest.mark.parametrize("n,m,l,k", [(5000, 24, 2, 1001), (3000, 96, 1, 2999), (2100, 7, 3, 2100)])
def test_topk_queries_any_k(n, m, l, k):
    """oracle_auto_topk accepts any k <= n (evaluate.py:43-46): k > 1000 runs the full-sort
    kernel; ids and fp64 distances equal the oracle's, ties (integer data) by id."""
    rng = np.random.default_rng(n)
    X = rng.integers(0, 5, (n, m)).astype(np.float32) if l == 3 else \
        rng.standard_normal((n, m)).astype(np.float32)
    A = rng.integers(1, 4, (n, l)).astype(np.int32)
    QX = rng.standard_normal((5, m))
    QA = rng.integers(1, 4, (5, l))
    qm = rng.integers(0, 2, (5, l))
    cfg = sb.MetricConfig.manual(0.7, l)
    ids, dists = sb.oracle_auto_topk_batch(X, A, QX, QA, k, cfg, qm, return_dists=True)
    for i in range(5):
        wi, wd = O.oracle_auto_topk(X, A, QX[i], QA[i], k, 0.7, qm[i], return_dists=True)
        np.testing.assert_array_equal(ids[i], wi)
        np.testing.assert_array_equal(dists[i], wd)


@pytest.mark.parametrize("n,k", [(3000, 1500), (1100, 1100), (1030, 2000)])
def test_bf_nodes_any_k(n, k):
    """brute_force_topk with k > 1024 (quality_k is unbounded in BuildParams): full-sort
    kernel, self excluded, -1 padding past n - 1 (_kernels.py:187,202-203)."""
    rng = np.random.default_rng(k)
    X = rng.integers(0, 3, (n, 5)).astype(np.float32)  # many exact ties
    A = rng.integers(1, 3, (n, 1)).astype(np.int32)
    s = np.sort(rng.choice(n, 9, replace=False)).astype(np.int64)
    got = DeviceIndex(X, A, 2).bf_topk_nodes(s, k, 0.45)
    want = O.kernels.brute_force_topk(X, A, 0.45, s, k)
    np.testing.assert_array_equal(got, want)


def test_hybrid_groundtruth_on_device():
    """oracle_hybrid_groundtruth (evaluate.py:58-77): exact-match filter (masked), pure feature
    distance, ties by id, fewer than k when matches are scarce, empty when none match."""
    rng = np.random.default_rng(3)
    n, m, l = 20000, 32, 3
    X = rng.integers(0, 3, (n, m)).astype(np.float32)
    A = rng.integers(1, 6, (n, l)).astype(np.int32)
    QX = rng.integers(0, 3, (30, m)).astype(np.float32)
    QA = rng.integers(1, 6, (30, l)).astype(np.int32)
    QA[0] = [9, 9, 9]          # no match
    masks = rng.integers(0, 2, (30, l))
    masks[1] = 0               # everything matches
    for k in (10, 200):
        got = sb.evaluate.oracle_hybrid_groundtruth_batch(X, A, QX, QA, k, masks)
        for i in range(30):
            want = O.oracle_hybrid_groundtruth(X, A, QX[i], QA[i], k, masks[i])
            np.testing.assert_array_equal(got[i], want, err_msg=f"query {i} k={k}")
            one = sb.oracle_hybrid_groundtruth(X, A, QX[i], QA[i], k, mask=masks[i])
            np.testing.assert_array_equal(one, want)
    assert got[0].size == 0


def test_search_results_survive_later_calls(small_golden):
    """Arrays returned by search() live in recycled page-locked blocks; a block may only be
    reused once no array (or row view) refers to it (returned views kept their
    block alive only through the wrong object)."""
    import gc
    gd = small_golden
    graph = sb.RelationGraph(features=gd["features"], attrs=gd["attrs"],
                             schema=sb.AttributeSchema(tuple(("x",) for _ in range(3))),
                             metric=sb.MetricConfig.manual(float(gd["alpha"]), 3), sigma=0.44,
                             nbr_ids=gd["final_ids"], nbr_dists=gd["final_dists"],
                             nbr_counts=gd["final_counts"], frozen=True)
    keep = []
    for qi in range(6):
        ids, dists, _ = sb.search(graph, gd["qf"][qi], gd["qa"][qi], sb.SearchParams(k=12), qi)
        keep.append((ids, dists, ids.copy(), dists.copy()))
        gc.collect()
    for ids, dists, ids0, dists0 in keep:
        np.testing.assert_array_equal(ids, ids0)
        np.testing.assert_array_equal(dists, dists0)


@pytest.mark.parametrize("kind", ["shell", "offset", "wide"])
def test_route_filter_near_ties_exact(kind, monkeypatch):
    """The certified fp32 filter of real-valued routing (route.cu kModeF64Filt, SB_ROUTE_FILT=1;
    off by default) must never drop
    a row that can enter the result list: rows on a thin shell around the query (distances
    equal to ~1e-9 relative, below fp32 resolution), rows far from the origin (the query's
    rounding to fp32 dominates), and d = 960 (cfg 4's width).  Ids, fp64 distances and the
    SearchStats counters equal the oracle's and the unfiltered path's."""
    rng = np.random.default_rng({"shell": 1, "offset": 2, "wide": 3}[kind])
    n, g, l = 3000, 16, 2
    m = 960 if kind == "wide" else 36
    q = 24
    qf = rng.standard_normal((q, m))
    if kind == "shell":
        dirs = rng.standard_normal((n, m))
        dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
        f = (qf[0] + dirs * (1.0 + 1e-9 * rng.integers(0, 50, (n, 1)))).astype(np.float32)
        qf = np.repeat(qf[:1], q, axis=0) + 1e-7 * rng.standard_normal((q, m))
    elif kind == "offset":
        f = (3e4 + rng.standard_normal((n, m))).astype(np.float32)
        qf = 3e4 + rng.standard_normal((q, m))
    else:
        f = rng.gamma(2.0, 1.0, (n, m)).astype(np.float32)
        qf = rng.gamma(2.0, 1.0, (q, m))
    a = rng.integers(1, 3, (n, l)).astype(np.int32)
    qa = rng.integers(1, 3, (q, l)).astype(np.int32)
    ids = np.stack([rng.choice(n, g, replace=False) for _ in range(n)]).astype(np.int32)
    cnt = rng.integers(g // 2, g + 1, n).astype(np.int32)
    graph = sb.RelationGraph(features=f, attrs=a, schema=sb.AttributeSchema((("x", "y"),) * l),
                             metric=sb.MetricConfig.manual(0.8, l), sigma=0.44, nbr_ids=ids,
                             nbr_dists=np.zeros((n, g), np.float32), nbr_counts=cnt, frozen=True)
    for k in (5, 64):
        p = sb.SearchParams(k=k, seed=4)
        monkeypatch.setenv("SB_ROUTE_FILT", "1")
        got = sb.search_batch_arrays(graph, qf, qa, p)
        assert graph.device().route_info()["path"] == "fp32-filter+fp64"
        monkeypatch.delenv("SB_ROUTE_FILT")
        plain = sb.search_batch_arrays(graph, qf, qa, p)
        assert graph.device().route_info()["path"] == "fp64"
        want = O.search_batch(f, a, ids, cnt, 0.8, qf, qa, k, seed=4)
        for x, y, z in zip(got, plain, want):
            np.testing.assert_array_equal(x[:, :z.shape[1]] if x.ndim == 2 else x, z, err_msg=f"{kind} k={k}")
            np.testing.assert_array_equal(x, y)

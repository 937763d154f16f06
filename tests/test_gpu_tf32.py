"""Exhaustive AUTO top-k for real-valued data on the tensor cores (bf_tf.cu): the TF32 filter
with a certified error bound must hand the exact re-rank every true member, so ids and fp64
distances equal the exact fp64 SIMT kernel and the CPU oracle (oracle_auto_topk,
evaluate.py:32-55) bit for bit — ragged K chunks, streamed and resident query tiles, masks,
duplicate points (ties by id), k up to 100, and queries whose candidates overflow the buffers
(recomputed on the fp64 kernel)."""

import os

import numpy as np
import pytest

import paper_2604_01617_b200 as sb
from oracle import oracle as O
from paper_2604_01617_b200.device import DeviceIndex

pytestmark = pytest.mark.gpu


def _data(kind, n, m, q, rng):
    if kind == "normal":
        f = rng.standard_normal((n, m)).astype(np.float32)
        qf = rng.standard_normal((q, m))
    elif kind == "gauss_w":  # cfg 5's recipe: N(0, I) W
        w = rng.standard_normal((m, m))
        f = (rng.standard_normal((n, m)) @ w).astype(np.float32)
        qf = (rng.standard_normal((q, m)) @ w).astype(np.float32).astype(np.float64)
    elif kind == "unit":  # cfg 3's recipe: clustered unit vectors
        mu = rng.standard_normal((16, m))
        mu /= np.linalg.norm(mu, axis=1, keepdims=True)
        x = 8.0 * mu[rng.integers(0, 16, n + q)] + rng.standard_normal((n + q, m))
        x = (x / np.linalg.norm(x, axis=1, keepdims=True)).astype(np.float32)
        f, qf = x[:n], x[n:].astype(np.float64)
    elif kind == "gamma":  # cfg 4's recipe: Gamma(2, 1) with a per-dimension scale
        s = np.exp(rng.uniform(-1, 1, m))
        f = (rng.gamma(2.0, 1.0, (n, m)) * s).astype(np.float32)
        qf = (rng.gamma(2.0, 1.0, (q, m)) * s).astype(np.float32).astype(np.float64)
    elif kind == "dup":  # duplicates and near-duplicates
        f = rng.standard_normal((n, m)).astype(np.float32)
        f[10:40] = f[3]
        f[50:60] = f[3] + np.float32(1e-6)
        qf = rng.standard_normal((q, m))
        qf[0] = f[3]
        qf[1] = f[3] + 1e-7
    else:
        raise ValueError(kind)
    return f, np.ascontiguousarray(qf, np.float64)


def _fp64_path(d, qf, qa, k, alpha, mk):
    os.environ["SB_BF_TF"] = "0"
    try:
        out = d.bf_topk_queries(qf, qa, k, alpha, mk)
        assert d.bf_info()["path"] == "fp64"
        return out
    finally:
        del os.environ["SB_BF_TF"]


@pytest.mark.parametrize("kind,n,m,l,q,k", [
    ("normal", 10000, 32, 1, 200, 10),     # cfg 1 shape
    ("gauss_w", 6000, 100, 1, 130, 10),    # d = 100: ragged last K chunk (104)
    ("unit", 3001, 96, 2, 129, 100),       # k = 100, ragged node and query tiles
    ("gamma", 2500, 960, 2, 70, 10),       # d = 960: streamed query tile
    ("normal", 777, 7, 3, 5, 1),           # d = 7, k = 1
    ("dup", 5000, 33, 2, 300, 32),         # ties by id
    ("unit", 20000, 96, 1, 300, 64),       # k > 32: two-pass bound (per-thread lists + select)
    ("gauss_w", 8000, 100, 1, 150, 250),   # two-pass, k = 250
    ("dup", 6000, 32, 2, 100, 600),        # two-pass with ties; fp64 check path = full sort
])
def test_tf32_topk_exact(kind, n, m, l, q, k):
    rng = np.random.default_rng(n + m + k)
    f, qf = _data(kind, n, m, q, rng)
    a = rng.integers(1, 5, (n, l)).astype(np.int32)
    qa = rng.integers(1, 5, (q, l))
    masks = rng.integers(0, 2, (q, l))
    alpha = 0.37 if kind != "unit" else 0.05
    d = DeviceIndex(f, a, 2)
    assert not d.info()["int_exact"]
    for mk in (None, masks):
        ids, dd = d.bf_topk_queries(qf, qa, k, alpha, mk)
        info = d.bf_info()
        assert info["path"] == "tc-tf32-filter", info
        assert info["fallback_queries"] == 0, info
        ids_s, dd_s = _fp64_path(d, qf, qa, k, alpha, mk)
        np.testing.assert_array_equal(ids, ids_s)
        np.testing.assert_array_equal(dd, dd_s)
        for qi in sorted(set(list(range(0, q, max(1, q // 6))) + [0, 1, q - 1])):
            wi, wd = O.oracle_auto_topk(f, a, qf[qi], qa[qi], k, alpha,
                                        None if mk is None else mk[qi], return_dists=True)
            np.testing.assert_array_equal(ids[qi], wi, err_msg=f"query {qi}")
            np.testing.assert_array_equal(dd[qi], wd, err_msg=f"query {qi}")


def test_tf32_filter_is_selective():
    """The certified window passes few candidates per query to the exact re-rank."""
    rng = np.random.default_rng(5)
    n, m, q, k = 20000, 96, 256, 10
    f, qf = _data("unit", n, m, q, rng)
    a = rng.integers(1, 4, (n, 1)).astype(np.int32)
    qa = rng.integers(1, 4, (q, 1))
    d = DeviceIndex(f, a, 2)
    d.bf_topk_queries(qf, qa, k, 0.2)
    info = d.bf_info()
    assert info["path"] == "tc-tf32-filter"
    assert info["candidates"] / q < 0.1 * n, info


@pytest.mark.parametrize("n", [3000, 12000])
def test_tf32_overflow_falls_back_exactly(n):
    """Points closer together than the TF32 window (steps of 1e-7 along one dimension): every
    node is a candidate, so the survivors overflow the re-rank (more than 2048); those queries
    are recomputed on the exact fp64 kernel and the answer is still the oracle's."""
    rng = np.random.default_rng(n)
    f = np.tile(rng.standard_normal((1, 40)).astype(np.float32), (n, 1))
    f[:, 0] += (np.arange(n) * 1e-7).astype(np.float32)
    a = np.ones((n, 1), np.int32)
    qf = rng.standard_normal((3, 40))
    qa = np.ones((3, 1), np.int64)
    d = DeviceIndex(f, a, 2)
    ids, dd = d.bf_topk_queries(qf, qa, 10, 0.5)
    info = d.bf_info()
    assert info["path"] == "tc-tf32-filter" and info["fallback_queries"] == 3, info
    for qi in range(3):
        wi, wd = O.oracle_auto_topk(f, a, qf[qi], qa[qi], 10, 0.5, return_dists=True)
        np.testing.assert_array_equal(ids[qi], wi)
        np.testing.assert_array_equal(dd[qi], wd)


def test_tf32_public_api_and_config_cfg1():
    """oracle_auto_topk_batch (the public API) on the cfg 1 recipe takes the TF32 path."""
    rng = np.random.default_rng(0)
    X = rng.standard_normal((10000, 32), dtype=np.float32)
    A = rng.integers(1, 5, (10000, 1), dtype=np.int32)
    QX = rng.standard_normal((200, 32), dtype=np.float32)
    QA = rng.integers(1, 5, (200, 1), dtype=np.int32)
    cfg = sb.compute_alpha(sb.sample_statistics(X, A, 1000, seed=0), 10000, 1)
    gt, gd = sb.oracle_auto_topk_batch(X, A, QX, QA, 10, cfg, return_dists=True)
    for qi in range(0, 200, 9):
        wi, wd = O.oracle_auto_topk(X, A, QX[qi], QA[qi], 10, cfg.alpha, return_dists=True)
        np.testing.assert_array_equal(gt[qi], wi)
        np.testing.assert_array_equal(gd[qi], wd)


@pytest.mark.parametrize("tile", ["128,4,1,2", "256,3,1,1", "128,3,1,1", "256,2,0,1", "128,4,0,1"])
def test_tf32_every_tile_shape(tile, monkeypatch):
    """Every kernel instance (two resident query tiles x 128 nodes; one query tile x 256 or 128
    nodes, resident or streamed) gives the exact answer, seed pass included."""
    monkeypatch.setenv("SB_TF_TILE", tile)
    rng = np.random.default_rng(7)
    n, m, l, q, k = 7000, 100, 2, 300, 16
    f, qf = _data("gauss_w", n, m, q, rng)
    a = rng.integers(1, 4, (n, l)).astype(np.int32)
    qa = rng.integers(1, 4, (q, l))
    masks = rng.integers(0, 2, (q, l))
    d = DeviceIndex(f, a, 2)
    ids, dd = d.bf_topk_queries(qf, qa, k, 0.6, masks)
    assert d.bf_info()["path"] == "tc-tf32-filter" and d.bf_info()["fallback_queries"] == 0
    ids_s, dd_s = _fp64_path(d, qf, qa, k, 0.6, masks)
    np.testing.assert_array_equal(ids, ids_s)
    np.testing.assert_array_equal(dd, dd_s)


@pytest.mark.parametrize("case", ["one_query", "zero_mask", "large_scale", "tiny_scale", "k_equals_n"])
def test_tf32_edge_cases(case):
    """Edge cases of the TF32 path: a single query, all-zero masks (no attribute term),
    values at 1e6 and 1e-6 scale (the certified margin scales with |x|^2 + |q|^2), and
    k = n (beyond the tensor-core list sizes: the exact fp64 kernel answers)."""
    rng = np.random.default_rng(["one_query", "zero_mask", "large_scale", "tiny_scale", "k_equals_n"].index(case))
    n, m, l, q, k = 3000, 24, 2, 40, 10
    f = rng.standard_normal((n, m)).astype(np.float32)
    qf = rng.standard_normal((q, m))
    if case == "large_scale":
        f *= np.float32(1e6)
        qf *= 1e6
    if case == "tiny_scale":
        f *= np.float32(1e-6)
        qf *= 1e-6
    if case == "one_query":
        qf = qf[:1]
        q = 1
    if case == "k_equals_n":
        n, k = 200, 200
        f = f[:n]
    a = rng.integers(1, 4, (n, l)).astype(np.int32)
    qa = rng.integers(1, 4, (q, l))
    mk = np.zeros((q, l), np.int64) if case == "zero_mask" else None
    d = DeviceIndex(f, a, 2)
    ids, dd = d.bf_topk_queries(qf, qa, k, 0.7, mk)
    if case != "k_equals_n":
        assert d.bf_info()["path"] == "tc-tf32-filter"
    for qi in range(q):
        wi, wd = O.oracle_auto_topk(f, a, qf[qi], qa[qi], k, 0.7, None if mk is None else mk[qi],
                                    return_dists=True)
        np.testing.assert_array_equal(ids[qi], wi, err_msg=f"{case} query {qi}")
        np.testing.assert_array_equal(dd[qi], wd, err_msg=f"{case} query {qi}")


def test_tf32_two_pass_equals_single_pass(monkeypatch):
    """k > 32: the two-pass bound (bf_tf.cu "large k") and the single pass with shared-memory
    lists (SB_TF_TWOPASS=0) give the reference's answer; the two-pass bound emits fewer
    candidates."""
    rng = np.random.default_rng(9)
    f, qf = _data("unit", 30000, 96, 400, rng)
    a = rng.integers(1, 4, (30000, 1)).astype(np.int32)
    qa = rng.integers(1, 4, (400, 1))
    d = DeviceIndex(f, a, 2)
    ids2, dd2 = d.bf_topk_queries(qf, qa, 100, 0.2)
    c2 = d.bf_info()["candidates"]
    monkeypatch.setenv("SB_TF_TWOPASS", "0")
    ids1, dd1 = d.bf_topk_queries(qf, qa, 100, 0.2)
    c1 = d.bf_info()["candidates"]
    np.testing.assert_array_equal(ids1, ids2)
    np.testing.assert_array_equal(dd1, dd2)
    assert c2 < c1, (c2, c1)


@pytest.mark.parametrize("m,k,scale", [(96, 10, 1.0), (96, 50, 1024.0), (960, 10, 1.0), (960, 32, 2.0 ** -20)])
def test_tf32_margin_adversarial(m, k, scale):
    """Worst case for the certified TF32 margin (bf_tf.cu tf_margin): every coordinate of the
    query and of its true neighbours sits just below a TF32 rounding midpoint
    (1 + 2^-11 - 2^-19 (1 + r)), so each operand loses almost 2^-11 in the same direction, x is
    parallel to q and |x| = |q| (both inequalities of the bound are tight): the filter sees
    S~ ~ 2^-10 (|x|^2 + |q|^2) for neighbours whose true S is ~1e-9 d, about 0.8 of the margin.
    The decoys are TF32-exact vectors (no operand error) that are truly farther but look four
    times nearer to the filter.  The exact top-k must still be the true neighbours: a margin
    below the real error would drop them silently."""
    rng = np.random.default_rng(m + k)
    n, l, q = 4000, 1, 8
    base = np.float32(1.0 + 2.0 ** -11 - 2.0 ** -19)
    qf32 = np.full((q, m), base, np.float32)
    qf32 -= (np.float32(2.0 ** -19) * rng.integers(0, 4, (q, m))).astype(np.float32)
    f = np.empty((n, m), np.float32)
    n_true = 3 * k
    f[:n_true] = base - (np.float32(2.0 ** -19) * rng.integers(0, 60, (n_true, m))).astype(np.float32)
    f[n_true:] = (1.0 + 2.0 ** -10 * rng.integers(0, 2, (n - n_true, m)) *
                  (rng.random((n - n_true, 1)) < 0.02)).astype(np.float32)  # sparse steps: near 1
    perm = rng.permutation(n)
    f = np.ascontiguousarray(f[perm] * np.float32(scale))
    qf = (qf32 * np.float32(scale)).astype(np.float64)
    a = np.ones((n, l), np.int32)
    qa = np.ones((q, l), np.int32)
    d = DeviceIndex(f, a, 2)
    ids, dd = d.bf_topk_queries(qf, qa, k, 0.7, None)
    assert d.bf_info()["path"] == "tc-tf32-filter"
    true_ids = set(np.nonzero(perm < n_true)[0].tolist())
    for qi in range(q):
        wi, wd = O.oracle_auto_topk(f, a, qf[qi], qa[qi], k, 0.7, return_dists=True)
        assert set(wi.tolist()) <= true_ids  # the construction: the exact answer is all true neighbours
        np.testing.assert_array_equal(ids[qi], wi, err_msg=f"query {qi}")
        np.testing.assert_array_equal(dd[qi], wd, err_msg=f"query {qi}")

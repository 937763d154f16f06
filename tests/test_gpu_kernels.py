"""GPU: the kernel-level drop-in (paper_2604_01617_b200._kernels) against the oracle's
restatement of hybridann._kernels, function by function, on identical inputs — including
the in-place mutation of adjacency / in-degree arrays — plus stress cases for the exact
overflow path of reinforce_pass."""

import numpy as np
import pytest

from paper_2604_01617_b200 import _kernels as G
from oracle import oracle as O
from paper_2604_01617_b200.device import DeviceIndex

pytestmark = pytest.mark.gpu


def _data(n, d, l, card, seed):
    rng = np.random.default_rng(seed)
    f = rng.standard_normal((n, d), dtype=np.float32)
    a = rng.integers(1, card + 1, (n, l), dtype=np.int32)
    s_v, s_a = O.sample_statistics(f, a, min(500, n), 0)
    return f, a, O.compute_alpha(s_v, s_a, n, l)


def test_compute_row_distances_and_candidates(small_golden):
    gd = small_golden
    f, a, alpha = gd["features"], gd["attrs"], float(gd["alpha"])
    rng = np.random.default_rng(0)
    ids = np.stack([rng.choice(np.delete(np.arange(600), i), 24, replace=False) for i in range(600)]).astype(np.int32)
    np.testing.assert_array_equal(G.compute_row_distances(f, a, ids, 1 / alpha),
                                  O.kernels.compute_row_distances(f, a, ids, 1 / alpha))
    fl_g = gd["it1_flags"].copy()
    fl_o = gd["it1_flags"].copy()
    got = G.build_candidates(gd["it1_ids"], fl_g, 24)
    want = O.kernels.build_candidates(gd["it1_ids"].copy(), fl_o, 24)
    for x, y in zip(got, want):
        np.testing.assert_array_equal(x, y)
    np.testing.assert_array_equal(fl_g, fl_o)
    for gn in (1, 7, 30):
        fl_g = gd["it1_flags"].copy()
        fl_o = gd["it1_flags"].copy()
        got = G.build_candidates(gd["it1_ids"], fl_g, gn)
        want = O.kernels.build_candidates(gd["it1_ids"].copy(), fl_o, gn)
        for x, y in zip(got, want):
            np.testing.assert_array_equal(x, y, err_msg=f"gamma_new={gn}")
        np.testing.assert_array_equal(fl_g, fl_o)


def test_local_join_in_place(small_golden):
    gd = small_golden
    f, a, alpha = gd["features"], gd["attrs"], float(gd["alpha"])
    for gn in (24, 9):
        st_o = [gd["init_ids"].copy(), gd["init_dists"].copy(), np.ones((600, 24), np.uint8)]
        st_g = [x.copy() for x in st_o]
        cand = O.kernels.build_candidates(st_o[0], st_o[2], gn)
        G.build_candidates(st_g[0], st_g[2], gn)
        ch_o = O.kernels.local_join(f, a, 1 / alpha, *cand, *st_o)
        ch_g = G.local_join(f, a, 1 / alpha, *cand, *st_g)
        assert (ch_o > 0) == (ch_g > 0)
        for x, y in zip(st_g, st_o):
            np.testing.assert_array_equal(x, y, err_msg=f"gamma_new={gn}")


def test_prune_reinforce_reconnect_in_place(overflow_golden):
    gd = overflow_golden
    f, a = gd["features"], gd["attrs"]
    last = int(gd["iterations"])
    n = f.shape[0]
    arrs_o = [gd[f"it{last}_ids"].copy(), gd[f"it{last}_dists"].copy(), np.full(n, 12, np.int32)]
    arrs_g = [x.copy() for x in arrs_o]
    indeg_o = O.kernels.count_in_degrees(arrs_o[0], arrs_o[2])
    indeg_g = G.count_in_degrees(arrs_g[0], arrs_g[2])
    np.testing.assert_array_equal(indeg_g, indeg_o)
    O.kernels.prune_pass(f, a, *arrs_o, indeg_o, 0.44)
    G.prune_pass(f, a, *arrs_g, indeg_g, 0.44)
    for x, y in zip(arrs_g + [indeg_g], arrs_o + [indeg_o]):
        np.testing.assert_array_equal(x, y)
    O.kernels.reinforce_pass(f, a, *arrs_o, indeg_o, 0.44)
    G.reinforce_pass(f, a, *arrs_g, indeg_g, 0.44)
    for x, y in zip(arrs_g + [indeg_g], arrs_o + [indeg_o]):
        np.testing.assert_array_equal(x, y)
    indeg_o = O.kernels.count_in_degrees(arrs_o[0], arrs_o[2])
    assert indeg_o.min() == 0, "case must exercise reconnect_islands"
    indeg_g = indeg_o.copy()
    O.kernels.reconnect_islands(f, a, *arrs_o, indeg_o, 0.44)
    G.reconnect_islands(f, a, *arrs_g, indeg_g, 0.44)
    for x, y in zip(arrs_g + [indeg_g], arrs_o + [indeg_o]):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("n,d,card,gamma,sigma,seed", [
    (2000, 16, 8, 16, 0.6, 5),      # thousands of full-row merges
    (1500, 16, 2, 12, 0.9, 5),      # nearly every row overflows
    (3000, 24, 3, 24, 0.44, 7),
    (2500, 40, 50, 32, 0.3, 11),    # high cardinality: cross-attribute rows never prune
])
def test_semantic_prune_overflow_stress(n, d, card, gamma, sigma, seed):
    f, a, alpha = _data(n, d, 1, card, seed)
    g = O.run_descent(f, a, alpha, gamma=gamma, gamma_new=gamma, seed=seed)
    base = (g.nbr_ids.copy(), g.nbr_dists.copy(), g.nbr_counts.copy())
    O.semantic_prune(g, sigma)
    import paper_2604_01617_b200 as sb
    from paper_2604_01617_b200.device import DeviceIndex
    dev = DeviceIndex(f, a, gamma)
    dev.upload(*base)
    dev.prune(sigma)
    over, sweeps = dev.reinforce(sigma)
    ids, dists, counts, _ = dev.download(with_flags=False)
    np.testing.assert_array_equal(counts, g.nbr_counts)
    np.testing.assert_array_equal(ids, g.nbr_ids)
    np.testing.assert_array_equal(dists, g.nbr_dists)
    assert sweeps == g.log["reconnect_sweeps"]


def test_bf_and_route_shim(small_golden):
    gd = small_golden
    f, a, alpha = gd["features"], gd["attrs"], float(gd["alpha"])
    s = gd["q_sample"]
    np.testing.assert_array_equal(G.brute_force_topk(f, a, 1 / alpha, s, 24),
                                  O.kernels.brute_force_topk(f, a, 1 / alpha, s, 24))
    assert G.graph_quality(gd["it1_ids"], np.full(600, 24, np.int32), s, gd["q_gt"]) == \
        O.kernels.graph_quality(gd["it1_ids"], np.full(600, 24, np.int32), s, gd["q_gt"])
    ids, cnt = gd["final_ids"], gd["final_counts"]
    for qi in range(0, 20, 3):
        qf = gd["qf"][qi].astype(np.float64)
        qa = gd["qa"][qi].astype(np.float64)
        qm = gd["qm"][qi].astype(np.float64)
        for k in (1, 15, 60):
            ent = O.entry_points(600, k, 0, qi)
            got = G.route(f, a, ids, cnt, qf, qa, qm, 1 / alpha, ent, max(1, k // 2), True)
            want = O.kernels.route(f, a, ids, cnt, qf, qa, qm, 1 / alpha, ent, max(1, k // 2), True)
            np.testing.assert_array_equal(got[0], want[0])
            np.testing.assert_array_equal(got[1], want[1])
            assert got[2:] == want[2:]


@pytest.mark.gpu
@pytest.mark.parametrize("n,g,seed", [(150, 100, 0), (2000, 64, 3), (50000, 100, 7), (300, 256, 1)])
def test_device_random_init_equals_numpy(n, g, seed):
    """sb_init_random_ids + host redraw of repeated rows == init_random_ids (graph.py:120-129),
    and the reported consumption leaves the generator exactly where NumPy's draw does."""
    from paper_2604_01617_b200.graph import init_random_ids, init_random_rows_device
    rng = np.random.default_rng(seed)
    f = rng.standard_normal((n, 4)).astype(np.float32)
    a = np.ones((n, 1), np.int32)
    dev = DeviceIndex(f, a, g)
    from paper_2604_01617_b200.graph import restored_generator
    consumed32, buffered, bad = dev.init_random_ids(seed)
    ref = np.random.default_rng(seed)
    ref.integers(0, n - 1, size=(n, g), dtype=np.int64)
    mine = restored_generator(seed, consumed32, buffered)
    rs, ms = ref.bit_generator.state, mine.bit_generator.state
    assert rs["state"] == ms["state"] and rs["has_uint32"] == ms["has_uint32"]
    if rs["has_uint32"]:
        assert rs["uinteger"] == ms["uinteger"]
    np.testing.assert_array_equal(ref.integers(0, 1 << 40, 64), mine.integers(0, 1 << 40, 64))
    np.testing.assert_array_equal(ref.choice(n - 1, 7, replace=False), mine.choice(n - 1, 7, replace=False))
    init_random_rows_device(dev, n, g, seed)
    host = init_random_ids(n, g, seed)
    np.testing.assert_array_equal(dev.download(with_flags=False)[0], host)
    # the initial rows built from the device ids equal those built from the host ids
    dev.init_graph(None, 1.0)
    ref_dev = DeviceIndex(f, a, g)
    ref_dev.init_graph(host, 1.0)
    for x, y in zip(dev.download(), ref_dev.download()):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("u8", ["1", "0"])
@pytest.mark.parametrize("n,d,card,gamma,sigma,seed", [
    (3000, 32, 3, 24, 0.44, 3),     # integer data in [0, 255], clustered: many redundant pairs
    (2000, 64, 1, 16, 0.6, 9),      # one attribute value: every pair is tested
])
def test_prune_integer_rows_u8_path(u8, n, d, card, gamma, sigma, seed, monkeypatch):
    """Integer features in [0, 255]: semantic_prune's cosines from u8 rows (dp4a, exact integer
    dot products and norms) equal the reference's fp64 _diff_cosine decisions bit for bit,
    exact duplicate points (zero-length offsets, cosine 1) included; SB_PRUNE_U8=0 runs the
    fp64 kernel on the same data."""
    monkeypatch.setenv("SB_PRUNE_U8", u8)
    rng = np.random.default_rng(seed)
    centres = rng.uniform(0, 255, (40, d))
    f = np.clip(np.rint(centres[rng.integers(0, 40, n)] + rng.normal(0, 12, (n, d))), 0, 255)
    f = f.astype(np.float32)
    f[100:110] = f[7]  # exact duplicates
    a = rng.integers(1, card + 1, (n, 1)).astype(np.int32)
    alpha = 0.8
    g = O.run_descent(f, a, alpha, gamma=gamma, gamma_new=gamma, seed=seed)
    base = (g.nbr_ids.copy(), g.nbr_dists.copy(), g.nbr_counts.copy())
    O.semantic_prune(g, sigma)
    from paper_2604_01617_b200.device import DeviceIndex
    dev = DeviceIndex(f, a, gamma)
    assert dev.info()["int_exact"]
    dev.upload(*base)
    dev.prune(sigma)
    dev.reinforce(sigma)
    ids, dists, counts, _ = dev.download(with_flags=False)
    np.testing.assert_array_equal(counts, g.nbr_counts)
    np.testing.assert_array_equal(ids, g.nbr_ids)
    np.testing.assert_array_equal(dists, g.nbr_dists)


@pytest.mark.parametrize("warp", ["1", "0"])
def test_device_entry_points_equal_reference(rng_golden, warp, monkeypatch):
    """The device entry-point kernels (warp-parallel Floyd draws with jump-ahead, the
    shared-memory and global-scratch per-thread kernels) reproduce the reference's
    entry_points (router.py:42-45) on the golden (n, k, seed, qi) grid (NumPy's Floyd and
    tail-shuffle regimes), and NumPy itself on query batches, including k = n and k = 1."""
    from paper_2604_01617_b200.device import entry_points_device
    monkeypatch.setenv("SB_EP_WARP", warp)
    gd = rng_golden
    for key in gd.files:
        if key.startswith("ep_"):
            _, n, k, seed, qi = key.split("_")
            got = entry_points_device(int(n), int(k), int(seed), int(qi), 1)[0]
            np.testing.assert_array_equal(got, gd[key], err_msg=key)
        elif key.startswith("ephead_"):
            _, n, k, seed, qi = key.split("_")
            got = entry_points_device(int(n), int(k), int(seed), int(qi), 1)[0]
            np.testing.assert_array_equal(got[:256], gd[key], err_msg=key)
    for n, k in ((1000, 1000), (5000, 1), (1_000_000, 200), (9999, 4000), (2_000_000, 3000)):
        got = entry_points_device(n, k, 7, 123, 300)
        want = np.stack([np.random.default_rng(np.random.SeedSequence(entropy=(7, 123 + i))).choice(n, k, replace=False)
                         for i in range(300)])
        np.testing.assert_array_equal(got, want, err_msg=f"n={n} k={k}")

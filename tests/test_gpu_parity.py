"""GPU parity: every device stage vs the reference's golden vectors and the CPU oracle.

The device path computes AUTO distances with explicitly rounded fp64 operations in the
reference's order, so parity here is bit-exact (ids, f32 row distances, flags, counts, fp64
search distances, all SearchStats counters) — stricter than the north star's tolerance
(ids exact except ties within 1e-5 relative; distances within 1e-5 relative).
"""

import numpy as np
import pytest

import paper_2604_01617_b200 as sb
from paper_2604_01617_b200.device import DeviceIndex
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _dev_from_state(gd, ids, dists, counts, flags, gamma):
    d = DeviceIndex(gd["features"], gd["attrs"], gamma)
    d.upload(ids, dists, counts, flags)
    return d


def _stage_check(gd, gamma, seed, sigma):
    """Run each device stage from the golden input of that stage and compare its output."""
    f, a, alpha = gd["features"], gd["attrs"], float(gd["alpha"])
    n = f.shape[0]
    inv = 1.0 / alpha
    # init
    ids0 = sb.init_random_ids(n, gamma, seed)
    d = DeviceIndex(f, a, gamma)
    d.init_graph(ids0, inv)
    ids, dists, counts, flags = d.download()
    np.testing.assert_array_equal(ids, gd["init_ids"])
    np.testing.assert_array_equal(dists, gd["init_dists"])
    assert (counts == gamma).all() and (flags == 1).all()
    # psi ground truth (node-mode brute force)
    gt = d.bf_topk_nodes(gd["q_sample"], gamma, inv)
    np.testing.assert_array_equal(gt, gd["q_gt"])
    # descent iterations, each from the golden previous state
    prev = (gd["init_ids"], gd["init_dists"], np.ones_like(gd["init_ids"], dtype=np.uint8))
    for it in range(1, int(gd["iterations"]) + 1):
        dd = _dev_from_state(gd, prev[0], prev[1], np.full(n, gamma, np.int32), prev[2], gamma)
        nc, ncnt, oc, ocnt = dd.build_candidates(gamma, download=True)
        fl = prev[2].copy()
        w_nc, w_ncnt, w_oc, w_ocnt = O.kernels.build_candidates(prev[0].copy(), fl, gamma)
        np.testing.assert_array_equal(ncnt, w_ncnt)
        np.testing.assert_array_equal(ocnt, w_ocnt)
        np.testing.assert_array_equal(nc, w_nc)
        np.testing.assert_array_equal(oc, w_oc)
        ins, pairs = dd.local_join(inv)
        assert ins > 0
        ids, dists, counts, flags = dd.download()
        np.testing.assert_array_equal(ids, gd[f"it{it}_ids"], err_msg=f"iteration {it}")
        np.testing.assert_array_equal(dists, gd[f"it{it}_dists"], err_msg=f"iteration {it}")
        np.testing.assert_array_equal(flags, gd[f"it{it}_flags"], err_msg=f"iteration {it}")
        prev = (ids, dists, flags)
    # prune from the golden post-descent state
    last = int(gd["iterations"])
    dp = _dev_from_state(gd, gd[f"it{last}_ids"], gd[f"it{last}_dists"],
                         np.full(n, gamma, np.int32), None, gamma)
    np.testing.assert_array_equal(dp.count_in_degrees(), gd["indeg0"])
    dp.prune(sigma)
    ids, dists, counts, _ = dp.download(with_flags=False)
    np.testing.assert_array_equal(counts, gd["prune_counts"])
    np.testing.assert_array_equal(ids, gd["prune_ids"])
    np.testing.assert_array_equal(dists, gd["prune_dists"])
    over, sweeps = dp.reinforce(sigma)
    ids, dists, counts, _ = dp.download(with_flags=False)
    np.testing.assert_array_equal(counts, gd["final_counts"])
    np.testing.assert_array_equal(ids, gd["final_ids"])
    np.testing.assert_array_equal(dists, gd["final_dists"])
    assert sweeps == int(gd["reconnect_sweeps"])
    return over


def test_small_every_stage(small_golden):
    _stage_check(small_golden, 24, 3, float(small_golden["sigma"]))


def test_overflow_every_stage(overflow_golden):
    over = _stage_check(overflow_golden, 12, 9, float(overflow_golden["sigma"]))
    assert over > 0, "case must take the exact sequential reinforce path"


def _graph(gd, gamma):
    return sb.RelationGraph(features=gd["features"], attrs=gd["attrs"],
                            schema=sb.AttributeSchema(tuple(("x",) for _ in range(gd["attrs"].shape[1]))),
                            metric=sb.MetricConfig.manual(float(gd["alpha"]), gd["attrs"].shape[1]),
                            sigma=0.44, nbr_ids=gd["final_ids"], nbr_dists=gd["final_dists"],
                            nbr_counts=gd["final_counts"], frozen=True)


def _check_search_keys(gd, graph, qf, qa, masks, prefix):
    keys = sorted(k for k in gd.files if k.startswith(prefix) and k.endswith("_ids"))
    assert keys
    for key in keys:
        tag = key[len(prefix):-len("_ids")]
        k = int(tag.split("_")[0][1:])
        coarse = tag.endswith("_c")
        ids, dists, st = sb.search_batch_arrays(graph, qf, qa, sb.SearchParams(k=k, use_coarse=coarse),
                                                masks=masks)
        np.testing.assert_array_equal(ids, gd[key], err_msg=key)
        np.testing.assert_array_equal(dists, gd[f"{prefix}{tag}_dists"], err_msg=key)
        np.testing.assert_array_equal(st[:, :4], gd[f"{prefix}{tag}_stats"], err_msg=key)


def test_small_searches_bit_exact(small_golden):
    gd = small_golden
    g = _graph(gd, 24)
    _check_search_keys(gd, g, gd["qf"], gd["qa"], gd["qm"], "s_")
    _check_search_keys(gd, g, gd["qf"], gd["qa"], None, "nomask_s_")


def test_single_search_equals_batch(small_golden):
    gd = small_golden
    g = _graph(gd, 24)
    ids, dists, stats = sb.search_batch(g, gd["qf"], gd["qa"], sb.SearchParams(k=15, seed=1),
                                        masks=gd["qm"])
    for qi in (0, 5, 19):
        one = sb.search(g, gd["qf"][qi], gd["qa"][qi], sb.SearchParams(k=15, seed=1, mask=gd["qm"][qi]), qi)
        np.testing.assert_array_equal(one[0], ids[qi])
        np.testing.assert_array_equal(one[1], dists[qi])
        assert one[2] == stats[qi]


def test_overflow_searches_bit_exact(overflow_golden):
    gd = overflow_golden
    _check_search_keys(gd, _graph(gd, 12), gd["qf"], gd["qa"], None, "s_")


def test_oracle_topk_matches_reference(small_golden):
    gd = small_golden
    cfg = sb.MetricConfig.manual(float(gd["alpha"]), 3)
    ids, dists = sb.oracle_auto_topk_batch(gd["features"], gd["attrs"], gd["qf"], gd["qa"], 20, cfg,
                                           gd["qm"], return_dists=True)
    np.testing.assert_array_equal(ids, gd["oracle_top20"])
    for qi in range(gd["qf"].shape[0]):
        wi, wd = O.oracle_auto_topk(gd["features"], gd["attrs"], gd["qf"][qi], gd["qa"][qi], 20,
                                    float(gd["alpha"]), gd["qm"][qi], return_dists=True)
        np.testing.assert_array_equal(dists[qi], wd)


def test_oracle_topk_tie_break_and_k_equals_n():
    f = np.zeros((5, 2), np.float32)
    a = np.ones((5, 1), np.int32)
    cfg = sb.MetricConfig.manual(1.0, 1)
    got = sb.oracle_auto_topk(f, a, np.ones(2, np.float32), [1], 5, cfg)
    np.testing.assert_array_equal(got, [0, 1, 2, 3, 4])
    with pytest.raises(ValueError):
        sb.oracle_auto_topk(f, a, np.ones(2, np.float32), [1], 6, cfg)


def test_bf_nodes_pads_when_n_small():
    rng = np.random.default_rng(0)
    f = rng.standard_normal((7, 3)).astype(np.float32)
    a = rng.integers(1, 3, (7, 1)).astype(np.int32)
    d = DeviceIndex(f, a, 2)
    got = d.bf_topk_nodes(np.array([0, 3, 6]), 10, 0.5)
    want = O.kernels.brute_force_topk(f, a, 0.5, np.array([0, 3, 6]), 10)
    np.testing.assert_array_equal(got, want)
    assert (got[:, 6:] == -1).all()


def test_bf_nodes_random_vs_oracle():
    rng = np.random.default_rng(1)
    for n, m, l, k in ((3000, 24, 2, 50), (5000, 100, 1, 100), (2000, 7, 3, 5), (1500, 256, 1, 64)):
        f = rng.standard_normal((n, m)).astype(np.float32)
        a = rng.integers(1, 4, (n, l)).astype(np.int32)
        s = np.sort(rng.choice(n, 37, replace=False)).astype(np.int64)
        got = DeviceIndex(f, a, 2).bf_topk_nodes(s, k, 0.37)
        want = O.kernels.brute_force_topk(f, a, 0.37, s, k)
        np.testing.assert_array_equal(got, want)


def test_route_random_graph_vs_oracle():
    """Routing on an arbitrary (non-HELP) graph, odd dims, masks, K=1..K=300."""
    rng = np.random.default_rng(2)
    n, m, l, g = 4000, 20, 3, 16
    f = rng.integers(0, 6, (n, m)).astype(np.float32)  # many exact ties
    a = rng.integers(1, 4, (n, l)).astype(np.int32)
    ids = np.stack([rng.choice(n, g, replace=False) for _ in range(n)]).astype(np.int32)
    cnt = rng.integers(1, g + 1, n).astype(np.int32)
    dists = np.zeros((n, g), np.float32)
    graph = sb.RelationGraph(features=f, attrs=a, schema=sb.AttributeSchema((("x",),) * l),
                             metric=sb.MetricConfig.manual(0.8, l), sigma=0.44, nbr_ids=ids,
                             nbr_dists=dists, nbr_counts=cnt, frozen=True)
    q = 64
    qf = rng.integers(0, 6, (q, m)).astype(np.float32)
    qa = rng.integers(1, 4, (q, l)).astype(np.int32)
    masks = rng.integers(0, 2, (q, l)).astype(np.float64)
    for k, coarse in ((1, True), (2, True), (7, False), (33, True), (300, True)):
        got = sb.search_batch_arrays(graph, qf, qa, sb.SearchParams(k=k, seed=5, use_coarse=coarse),
                                     masks=masks)
        want = O.search_batch(f, a, ids, cnt, 0.8, qf, qa, k, seed=5, masks=masks, use_coarse=coarse)
        np.testing.assert_array_equal(got[0], want[0], err_msg=f"k={k}")
        np.testing.assert_array_equal(got[1], want[1], err_msg=f"k={k}")
        np.testing.assert_array_equal(got[2][:, :4], want[2], err_msg=f"k={k}")


@pytest.mark.parametrize("relabel", ["1", "0"])
@pytest.mark.parametrize("g,path", [(32, "u8"), (24, "fp32"), (16, "fp64")])
def test_route_large_k_insertion_buffer(relabel, g, path, monkeypatch):
    """K >= 512 routes through the insertion-buffer kernel instance (new candidates wait in a
    small sorted buffer next to the K-list); every result must equal the oracle bit for bit:
    ties everywhere (features in {0..3}), both phases, masks, relabeled layout or not, and the
    same answers as the plain instance (SB_ROUTE_LAZY=0)."""
    monkeypatch.setenv("SB_ROUTE_RELABEL", relabel)
    rng = np.random.default_rng(11 + g)
    n, m, l = 9000, 32, 2
    f = rng.integers(0, 4, (n, m)).astype(np.float32)
    if path == "fp64":
        f = f + np.float32(0.5) * rng.integers(0, 2, (n, m)).astype(np.float32) * np.float32(0.001)
    if path == "fp32":
        monkeypatch.setenv("SB_ROUTE_U8", "0")
    a = rng.integers(1, 4, (n, l)).astype(np.int32)
    ids = np.stack([rng.choice(n, g, replace=False) for _ in range(n)]).astype(np.int32)
    cnt = rng.integers(g // 2, g + 1, n).astype(np.int32)

    def graph():
        return sb.RelationGraph(features=f, attrs=a, schema=sb.AttributeSchema((("x",),) * l),
                                metric=sb.MetricConfig.manual(0.9, l), sigma=0.44, nbr_ids=ids,
                                nbr_dists=np.zeros((n, g), np.float32), nbr_counts=cnt, frozen=True)
    q = 24
    qf = rng.integers(0, 4, (q, m)).astype(np.float32)
    qa = rng.integers(1, 4, (q, l)).astype(np.int32)
    masks = rng.integers(0, 2, (q, l)).astype(np.float64)
    gr = graph()
    for k, coarse in ((600, True), (1000, False), (2500, True)):
        p = sb.SearchParams(k=k, seed=7, use_coarse=coarse)
        got = sb.search_batch_arrays(gr, qf, qa, p, masks=masks)
        want = O.search_batch(f, a, ids, cnt, 0.9, qf, qa, k, seed=7, masks=masks, use_coarse=coarse)
        np.testing.assert_array_equal(got[0], want[0], err_msg=f"k={k}")
        np.testing.assert_array_equal(got[1], want[1], err_msg=f"k={k}")
        np.testing.assert_array_equal(got[2][:, :4], want[2], err_msg=f"k={k}")
    want_path = {"u8": "u8-dp4a", "fp32": "fp32", "fp64": "fp64"}[path]
    assert gr.device().route_info()["path"] == want_path


@pytest.mark.parametrize("k,force", [(600, True), (2000, True), (17000, False)])
def test_route_result_list_in_global_memory(k, force, monkeypatch):
    """K beyond shared memory (cfg 5 at cardinality 10^4 needs K near 3·Θ):
    each slot's result list lives in global memory (automatic once it outgrows shared memory;
    SB_ROUTE_RGLOBAL=1 forces it for any K served by the large-K kernel instance).  Results equal the oracle bit for bit."""
    if force:
        monkeypatch.setenv("SB_ROUTE_RGLOBAL", "1")
    rng = np.random.default_rng(k)
    n, m, l, g = 24000 if k > 1000 else 6000, 24, 1, 20
    f = rng.integers(0, 5, (n, m)).astype(np.float32)
    a = rng.integers(1, 30, (n, l)).astype(np.int32)
    ids = np.stack([rng.choice(n, g, replace=False) for _ in range(n)]).astype(np.int32)
    cnt = rng.integers(g // 2, g + 1, n).astype(np.int32)
    gr = sb.RelationGraph(features=f, attrs=a, schema=sb.AttributeSchema((("x",),) * l),
                          metric=sb.MetricConfig.manual(0.7, l), sigma=0.44, nbr_ids=ids,
                          nbr_dists=np.zeros((n, g), np.float32), nbr_counts=cnt, frozen=True)
    q = 3 if k > 1000 else 20
    qf = rng.integers(0, 5, (q, m)).astype(np.float32)
    qa = rng.integers(1, 30, (q, l)).astype(np.int32)
    masks = rng.integers(0, 2, (q, l)).astype(np.float64)
    p = sb.SearchParams(k=k, seed=3, use_coarse=True)
    got = sb.search_batch_arrays(gr, qf, qa, p, masks=masks)
    want = O.search_batch(f, a, ids, cnt, 0.7, qf, qa, k, seed=3, masks=masks, use_coarse=True)
    np.testing.assert_array_equal(got[0], want[0])
    np.testing.assert_array_equal(got[1], want[1])
    np.testing.assert_array_equal(got[2][:, :4], want[2])


def test_order_free_mode_is_bit_exact():
    """Integer-valued data in [0, 255] routes through the u8/dp4a path by default; the fp32
    order-free paths (one row per lane, lane groups), the fp64 lane path and the sequential
    path must all equal the oracle bit for bit (ids, fp64 dists, all stats)."""
    rng = np.random.default_rng(3)
    n, m, l, g = 6000, 128, 3, 24
    f = np.clip(np.rint(rng.normal(128, 40, (n, m))), 0, 255).astype(np.float32)
    a = rng.integers(1, 6, (n, l)).astype(np.int32)
    ids = np.stack([rng.choice(n, g, replace=False) for _ in range(n)]).astype(np.int32)
    cnt = rng.integers(1, g + 1, n).astype(np.int32)
    graph = sb.RelationGraph(features=f, attrs=a, schema=sb.AttributeSchema((("x",),) * l),
                             metric=sb.MetricConfig.manual(1.03, l), sigma=0.44, nbr_ids=ids,
                             nbr_dists=np.zeros((n, g), np.float32), nbr_counts=cnt, frozen=True)
    dev = graph.device()
    assert dev.info()["int_exact"]
    qf = np.clip(np.rint(rng.normal(128, 40, (48, m))), 0, 255).astype(np.float32)
    qa = rng.integers(1, 6, (48, l)).astype(np.int32)
    import os
    def with_env(env, fn):
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            return fn()
        finally:
            for k, v in old.items():
                if v is None:
                    del os.environ[k]
                else:
                    os.environ[k] = v
    for k in (5, 64, 257):
        p = sb.SearchParams(k=k, seed=2)
        run = lambda: sb.search_batch_arrays(graph, qf, qa, p)
        u8 = run()
        assert dev.route_info()["path"] == "u8-dp4a"
        lane = with_env({"SB_ROUTE_U8": "0"}, run)
        assert dev.route_info()["path"] == "fp32"
        split = with_env({"SB_ROUTE_U8": "0", "SB_ROUTE_LPR": "8"}, run)
        f64 = with_env({"SB_ROUTE_F32": "0"}, run)
        assert dev.route_info()["path"] == "fp64"
        f64u = with_env({"SB_ROUTE_F32": "0", "SB_ROUTE_FILT": "1"}, run)
        assert dev.route_info()["path"] == "fp32-filter+fp64"
        dev.set_distance_mode(sequential=True)
        seq = sb.search_batch_arrays(graph, qf, qa, p)
        dev.set_distance_mode(sequential=False)
        want = O.search_batch(f, a, ids, cnt, 1.03, qf, qa, k, seed=2)
        for got in (u8, lane, split, f64, f64u, seq):
            np.testing.assert_array_equal(got[0], want[0])
            np.testing.assert_array_equal(got[1], want[1])
            np.testing.assert_array_equal(got[2][:, :4], want[2])
    # a non-integral query falls back to the sequential path, still exact
    qf2 = qf + 0.25
    got = sb.search_batch_arrays(graph, qf2, qa, sb.SearchParams(k=33))
    want = O.search_batch(f, a, ids, cnt, 1.03, qf2, qa, 33)
    np.testing.assert_array_equal(got[0], want[0])
    np.testing.assert_array_equal(got[1], want[1])
    # real-valued features never take the order-free path
    fr = f + np.float32(0.5)
    assert not sb.RelationGraph(features=fr, attrs=a, schema=graph.schema, metric=graph.metric,
                                sigma=0.44, nbr_ids=ids, nbr_dists=graph.nbr_dists,
                                nbr_counts=cnt, frozen=True).device().info()["int_exact"]


@pytest.mark.parametrize("n,m,l,q,k,lo", [(5000, 128, 3, 300, 10, 0), (3001, 64, 2, 129, 16, 0),
                                          (777, 32, 1, 5, 1, 0), (20000, 128, 3, 1000, 10, 0),
                                          (4000, 48, 2, 200, 10, -255)])
@pytest.mark.parametrize("path", ["u8", "bf16", "fold"])
def test_tensor_core_topk_exact(n, m, l, q, k, lo, path):
    """tcgen05 paths (integer data: u8 operands with kind::i8, bf16 operands, bf16 with |x|^2
    folded into the MMA): identical ids and fp64 distances to the fp64 SIMT path and to the
    oracle, including ragged tiles (n % 256, q % 128), masks, duplicate points and signed
    values (which take the bf16 path)."""
    import os
    os.environ["SB_BF_U8"] = "1" if path == "u8" else "0"
    os.environ["SB_BF_FOLD"] = "1" if path == "fold" else "0"
    rng = np.random.default_rng(n + m)
    f = np.clip(np.rint(rng.normal(128 + lo, 50 - lo / 3, (n, m))), lo, 255).astype(np.float32)
    f[10:20] = f[5]                      # exact duplicates: ties broken by id
    a = rng.integers(1, 6, (n, l)).astype(np.int32)
    qf = np.clip(np.rint(rng.normal(128 + lo, 50 - lo / 3, (q, m))), lo, 255)
    qf[0] = f[5]
    qa = rng.integers(1, 6, (q, l))
    masks = rng.integers(0, 2, (q, l))
    cfg = sb.MetricConfig.manual(0.91, l)
    d = DeviceIndex(f, a, 2)
    for mk in (None, masks):
        ids_tc, dd_tc = d.bf_topk_queries(qf, qa, k, cfg.alpha, mk)
        assert d.info()["last_bf_tc"], "tensor-core path not taken"
        os.environ["SB_BF_TC"] = "0"
        try:
            ids_s, dd_s = d.bf_topk_queries(qf, qa, k, cfg.alpha, mk)
            assert not d.info()["last_bf_tc"]
        finally:
            del os.environ["SB_BF_TC"]
        np.testing.assert_array_equal(ids_tc, ids_s)
        np.testing.assert_array_equal(dd_tc, dd_s)
        for qi in list(range(0, q, max(1, q // 7))) + [0]:
            wi, wd = O.oracle_auto_topk(f, a, qf[qi], qa[qi], k, cfg.alpha,
                                        None if mk is None else mk[qi], return_dists=True)
            np.testing.assert_array_equal(ids_tc[qi], wi)
            np.testing.assert_array_equal(dd_tc[qi], wd)
    del os.environ["SB_BF_FOLD"]
    del os.environ["SB_BF_U8"]


@pytest.mark.slow
def test_cfg1_end_to_end(cfg1_golden):
    """BASELINE config 1 through the public API: alpha, psi history, edge counts, final
    adjacency hashes, searches at K = 10 / 25 / 50 (ids, dists, stats) and the exact GT."""
    import hashlib
    gd = cfg1_golden

    def sha(x):
        x = np.ascontiguousarray(x)
        return hashlib.sha256(x.tobytes() + str(x.dtype).encode() + str(x.shape).encode()).hexdigest()

    rng = np.random.default_rng(0)
    X = rng.standard_normal((10000, 32), dtype=np.float32)
    A = rng.integers(1, 5, (10000, 1), dtype=np.int32)
    QX = rng.standard_normal((200, 32), dtype=np.float32)
    QA = rng.integers(1, 5, (200, 1), dtype=np.int32)
    cfg = sb.compute_alpha(sb.sample_statistics(X, A, 1000, seed=0), 10000, 1)
    assert cfg.alpha == float(gd["alpha"])
    g = sb.build(X, A, sb.AttributeSchema((("v1", "v2", "v3", "v4"),)), sb.BuildParams(), cfg)
    np.testing.assert_array_equal(np.array(g.build_log["psi_history"]), gd["psi_history"])
    assert sha(g.nbr_counts) == str(gd["sha_final_counts"])
    assert sha(g.nbr_ids) == str(gd["sha_final_ids"])
    assert sha(g.nbr_dists) == str(gd["sha_final_dists"])
    assert int(g.nbr_counts.sum()) == 194_468
    for k in (10, 25, 50):
        ids, dists, st = sb.search_batch_arrays(g, QX, QA, sb.SearchParams(k=k))
        np.testing.assert_array_equal(ids, gd[f"s_k{k}_c_ids"])
        np.testing.assert_array_equal(dists, gd[f"s_k{k}_c_dists"])
        np.testing.assert_array_equal(st[:, :4], gd[f"s_k{k}_c_stats"])
    gt = sb.oracle_auto_topk_batch(X, A, QX, QA, 10, cfg)
    np.testing.assert_array_equal(gt, gd["oracle_top10"])
    # recall at the operating point K=25 (0.9550)
    ids, _, _ = sb.search_batch_arrays(g, QX, QA, sb.SearchParams(k=25))
    assert sb.mean_recall(ids, gt, 10) == pytest.approx(0.955, abs=1e-9)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,n,q", [("cfg2", 3000, 40), ("cfg3", 3000, 40), ("cfg4", 1200, 20),
                                     ("cfg5c10", 3000, 40), ("cfg5c1", 2000, 30)])
def test_config_recipes_end_to_end(cfg, n, q):
    """Every BASELINE config recipe (tools/configs.py) at reduced N: the GPU HELP build equals
    the oracle's graph bit for bit, and GPU routing / exact top-k equal the oracle's."""
    from tools.configs import make_config
    X, A, QX, QA, card = make_config(cfg, n)
    QX, QA = QX[:q], QA[:q]
    cfg_m = sb.compute_alpha(sb.sample_statistics(X, A, min(1000, n), seed=0), n, A.shape[1])
    schema = sb.AttributeSchema(tuple(tuple(str(i) for i in range(c)) for c in card))
    p = sb.BuildParams(gamma=32, gamma_new=32)
    g = sb.build(X, A, schema, p, cfg_m)
    og = O.build(X, A, cfg_m.alpha, sigma=p.sigma, gamma=p.gamma, gamma_new=p.gamma_new)
    np.testing.assert_array_equal(g.nbr_counts, og.nbr_counts)
    for i in range(n):
        c = og.nbr_counts[i]
        np.testing.assert_array_equal(g.nbr_ids[i, :c], og.nbr_ids[i, :c])
        np.testing.assert_array_equal(g.nbr_dists[i, :c], og.nbr_dists[i, :c])
    for k in (10, 50):
        got = sb.search_batch_arrays(g, QX, QA, sb.SearchParams(k=k))
        want = O.search_batch(X, A, og.nbr_ids, og.nbr_counts, cfg_m.alpha, QX, QA, k)
        np.testing.assert_array_equal(got[0], want[0])
        np.testing.assert_array_equal(got[1], want[1])
        np.testing.assert_array_equal(got[2][:, :4], want[2])
    ti, td = sb.oracle_auto_topk_batch(X, A, QX, QA, 10, cfg_m, return_dists=True)
    for i in range(q):
        wi, wd = O.oracle_auto_topk(X, A, QX[i], QA[i], 10, cfg_m.alpha, return_dists=True)
        np.testing.assert_array_equal(ti[i], wi)
        np.testing.assert_array_equal(td[i], wd)


@pytest.mark.gpu
def test_route_layout_follows_adjacency_changes():
    """The relabeled routing layout is rebuilt when the adjacency changes, and routing with
    and without it (SB_ROUTE_RELABEL=0) equals the oracle."""
    import os
    rng = np.random.default_rng(11)
    n, m, l, g = 3000, 16, 2, 12
    f = rng.integers(0, 4, (n, m)).astype(np.float32)
    a = rng.integers(1, 3, (n, l)).astype(np.int32)
    qf = rng.integers(0, 4, (20, m)).astype(np.float32)
    qa = rng.integers(1, 3, (20, l)).astype(np.int32)
    dev = DeviceIndex(f, a, g)
    for trial in range(2):
        ids = np.stack([rng.choice(n, g, replace=False) for _ in range(n)]).astype(np.int32)
        cnt = rng.integers(1, g + 1, n).astype(np.int32)
        dev.upload(ids, np.zeros((n, g), np.float32), cnt)
        want = O.search_batch(f, a, ids, cnt, 0.9, qf, qa, 24, seed=1)
        ent = O.all_entry_points(n, 24, 1, qf.shape[0])
        for relabel in ("1", "0"):
            os.environ["SB_ROUTE_RELABEL"] = relabel
            try:
                got = dev.route(qf, qa, 24, 12, 1.0 / 0.9, entries=ent)
            finally:
                del os.environ["SB_ROUTE_RELABEL"]
            np.testing.assert_array_equal(got[0], want[0], err_msg=f"trial {trial} relabel {relabel}")
            np.testing.assert_array_equal(got[1], want[1])
            np.testing.assert_array_equal(got[2][:, :4], want[2])


def test_route_on_reference_written_index():
    """Routing over the graph the reference wrote (write_index) and read back (read_index),
    bit for bit against the reference's own searches of its read-back graph
    (tests/golden/make_golden.py case_index; graph.py:287-415, _kernels.py:504-610)."""
    import os
    gd = np.load(os.path.join(os.path.dirname(__file__), "golden", "index.npz"))
    g = sb.read_index(os.path.join(os.path.dirname(__file__), "golden", "small_index.help"))
    for k in (10, 30):
        ids, dists, st = sb.search_batch_arrays(g, gd["qf"], gd["qa"], sb.SearchParams(k=k))
        np.testing.assert_array_equal(ids, gd[f"s_k{k}_c_ids"])
        np.testing.assert_array_equal(dists, gd[f"s_k{k}_c_dists"])
        np.testing.assert_array_equal(st[:, :4], gd[f"s_k{k}_c_stats"])


def test_bench_sweep_matches_reference():
    """bench_sweep (evaluate.py:95-141) through the device: pioneer sizes, mean Recall@10 and
    mean distance evaluations equal the reference's own bench_sweep on the same graph and
    ground truth; the roofline columns equal §8(d)'s bytes from the search stats."""
    import os
    gd = np.load(os.path.join(os.path.dirname(__file__), "golden", "index.npz"))
    g = sb.read_index(os.path.join(os.path.dirname(__file__), "golden", "small_index.help"))
    gt = list(gd["sweep_gt"])
    rows = sb.evaluate.bench_sweep(g, gd["qf"], gd["qa"], gt, [5, 10, 30], timing_passes=2,
                                   hbm_peak_gbs=6500.0)
    for r, want in zip(rows, gd["sweep"]):
        assert (r.k, r.pioneer, r.n_queries) == (int(want[0]), int(want[1]), int(want[4]))
        assert r.mean_recall_at_10 == want[2] and r.mean_dist_evals == want[3]
        assert r.qps > 0 and r.algorithmic_gbs > 0
        assert abs(r.hbm_frac - r.algorithmic_gbs / 6500.0) < 1e-12
    _, _, st = sb.search_batch_arrays(g, gd["qf"], gd["qa"], sb.SearchParams(k=30))
    m, l = g.features.shape[1], g.attrs.shape[1]
    assert sb.evaluate.routing_bytes(st, m, l) == \
        float(st[:, 0].sum() * (4 * m + 4 * l) + 4 * (st[:, 2].sum() + st[:, 3].sum() + st[:, 4].sum()))


@pytest.mark.parametrize("deep", ["1", "0"])
@pytest.mark.parametrize("m,g,k", [(4, 16, 9), (36, 8, 40), (100, 40, 64), (132, 100, 200),
                                   (960, 24, 50), (64, 48, 1500)])
def test_route_real_valued_both_instances(deep, m, g, k, monkeypatch):
    """Real-valued rows (exact sequential fp64, _kernels.py:26-35) through both kernel instances:
    the staged one (cp.async row lines in a shared-memory ring, conversion-free fp32 -> fp64:
    small batches and long rows) and the three-CTA one (SB_ROUTE_DEEP=0).  Dimensions below,
    at and off whole 128-byte lines, batches above the ring's rows per round (g = 100), K in
    the insertion-buffer range, masks, subnormal / zero / huge features."""
    monkeypatch.setenv("SB_ROUTE_DEEP", deep)
    rng = np.random.default_rng(100 + m)
    n, l, q = 3000, 2, 48
    f = (rng.standard_normal((n, m)) * np.exp(rng.uniform(-3, 3, (1, m)))).astype(np.float32)
    f[rng.integers(0, n, 40), rng.integers(0, m, 40)] = 0.0
    f[rng.integers(0, n, 40), rng.integers(0, m, 40)] = np.float32(1e-41)   # subnormal
    f[rng.integers(0, n, 40), rng.integers(0, m, 40)] = np.float32(-3e-39)  # subnormal
    f[rng.integers(0, n, 10), rng.integers(0, m, 10)] = np.float32(1e18)
    a = rng.integers(1, 5, (n, l)).astype(np.int32)
    ids = np.stack([rng.choice(n, g, replace=False) for _ in range(n)]).astype(np.int32)
    cnt = rng.integers(max(1, g // 2), g + 1, n).astype(np.int32)
    graph = sb.RelationGraph(features=f, attrs=a, schema=sb.AttributeSchema((("x",),) * l),
                             metric=sb.MetricConfig.manual(0.7, l), sigma=0.44, nbr_ids=ids,
                             nbr_dists=np.zeros((n, g), np.float32), nbr_counts=cnt, frozen=True)
    qf = (rng.standard_normal((q, m)) * 2).astype(np.float32)
    qf[0] = f[7]          # a query equal to a node: zero differences
    qa = rng.integers(1, 5, (q, l)).astype(np.int32)
    masks = rng.integers(0, 2, (q, l)).astype(np.float64)
    for mk in (None, masks):
        got = sb.search_batch_arrays(graph, qf, qa, sb.SearchParams(k=k, seed=3), masks=mk)
        info = graph.device().route_info()
        assert info["path"] == "fp64" and info["pipelined"] == (deep == "1")
        want = O.search_batch(f, a, ids, cnt, 0.7, qf, qa, k, seed=3, masks=mk)
        np.testing.assert_array_equal(got[0], want[0])
        np.testing.assert_array_equal(got[1], want[1])
        np.testing.assert_array_equal(got[2][:, :4], want[2])

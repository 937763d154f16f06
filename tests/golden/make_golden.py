"""Generate golden vectors by running the CPU reference itself (hybridann 0.1.0).

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_golden python tests/golden/make_golden.py

The reference is imported read-only from /root/reference/pkg/src; its own
functions produce every array stored here.  Intermediate build states are
captured by driving the reference's public pieces in the same order as
graph.build / graph.semantic_prune (graph.py:202-280).  Fixtures are small
(.npz); the cfg-1 adjacency is pinned by SHA-256 of its arrays.

Cases
  small     reference conftest dataset (n=600, m=12, L=3, pool 3, seeds 11/12/13),
            Gamma=24 build seed 3, 20 queries (generate_queries seed 14): every
            stage's full arrays, searches over a K grid with masks, oracle GT.
  overflow  n=1500, d=32, L=1 card 4, Gamma=12: reinforce_pass overflows (375 full-row
            merges + re-prune) and one reconnect_islands sweep runs; full arrays per stage.
  cfg1      BASELINE config 1 (N=10k, d=32, card 4, 200 queries, seed 0, BuildParams()):
            alpha, psi history, edge counts, hashes of every stage, searches at
            K in {10, 25, 50} (ids, dists, stats) and the exact AUTO top-10 GT.
  index     the small case's graph written by the reference's write_index (small_index.help)
            and searched after the reference's read_index.
  rng       entry_points over an (n, K, seed, qi) grid covering NumPy's two
            choice() regimes; init_random_graph id matrices (pre-distance).
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes() + str(a.dtype).encode() + str(a.shape).encode()).hexdigest()


def staged_build(ha, features, attrs, schema, params, config):
    """graph.build split into stages (graph.py:235-280) with snapshots."""
    from hybridann import _kernels
    from hybridann.graph import (descent_iteration, estimate_graph_quality, init_random_graph,
                                 prepare_quality_estimate)
    st = {}
    g = init_random_graph(features, attrs, schema, params, config)
    st["init_ids"], st["init_dists"] = g.nbr_ids.copy(), g.nbr_dists.copy()
    q = prepare_quality_estimate(g, params)
    st["q_sample"], st["q_gt"] = q.sample_ids.copy(), q.ground_truth.copy()
    psi = [estimate_graph_quality(g, q)]
    it = 0
    changes_hist = []
    while psi[-1] < params.psi_target and it < params.max_iterations:
        ch = descent_iteration(g, params)
        it += 1
        changes_hist.append(ch)
        psi.append(estimate_graph_quality(g, q))
        st[f"it{it}_ids"], st[f"it{it}_dists"], st[f"it{it}_flags"] = (
            g.nbr_ids.copy(), g.nbr_dists.copy(), g.nbr_flags.copy())
        if ch == 0:
            break
    st["iterations"] = np.int64(it)
    st["psi_history"] = np.array(psi, np.float64)
    st["changes_nonzero"] = np.array([c > 0 for c in changes_hist])
    in_deg = _kernels.count_in_degrees(g.nbr_ids, g.nbr_counts)
    st["indeg0"] = in_deg.copy()
    _kernels.prune_pass(g.features, g.attrs, g.nbr_ids, g.nbr_dists, g.nbr_counts, in_deg, params.sigma)
    st["prune_ids"], st["prune_dists"], st["prune_counts"] = (
        g.nbr_ids.copy(), g.nbr_dists.copy(), g.nbr_counts.copy())
    st["prune_indeg"] = in_deg.copy()
    _kernels.reinforce_pass(g.features, g.attrs, g.nbr_ids, g.nbr_dists, g.nbr_counts, in_deg, params.sigma)
    st["reinf_ids"], st["reinf_dists"], st["reinf_counts"] = (
        g.nbr_ids.copy(), g.nbr_dists.copy(), g.nbr_counts.copy())
    sweeps = 0
    for _ in range(10):
        in_deg = _kernels.count_in_degrees(g.nbr_ids, g.nbr_counts)
        if in_deg.min() >= 1:
            break
        _kernels.reconnect_islands(g.features, g.attrs, g.nbr_ids, g.nbr_dists, g.nbr_counts,
                                   in_deg, params.sigma)
        sweeps += 1
    st["reconnect_sweeps"] = np.int64(sweeps)
    st["final_ids"], st["final_dists"], st["final_counts"] = (
        g.nbr_ids.copy(), g.nbr_dists.copy(), g.nbr_counts.copy())
    # cross-check: the staged pipeline equals the reference's own build()
    ref = ha.build(features, attrs, schema, params, config)
    assert np.array_equal(ref.nbr_ids, g.nbr_ids) and np.array_equal(ref.nbr_counts, g.nbr_counts)
    assert ref.build_log["psi_history"] == psi
    ref.frozen = True
    return st, ref


def searches(ha, graph, qf, qa, ks, masks=None, coarse=(True, False), seed=0):
    out = {}
    for k in ks:
        for uc in coarse:
            ids = np.empty((qf.shape[0], k), np.int64)
            dists = np.empty((qf.shape[0], k), np.float64)
            stats = np.empty((qf.shape[0], 4), np.int64)
            for qi in range(qf.shape[0]):
                p = ha.SearchParams(k=k, seed=seed, mask=None if masks is None else masks[qi],
                                    use_coarse=uc)
                i, d, s = ha.search(graph, qf[qi], qa[qi], p, qi)
                ids[qi], dists[qi] = i, d
                stats[qi] = (s.dist_evals, s.phase1_evals, s.phase1_expansions, s.hops)
            tag = f"k{k}_{'c' if uc else 'r'}"
            out[f"s_{tag}_ids"], out[f"s_{tag}_dists"], out[f"s_{tag}_stats"] = ids, dists, stats
    return out


def case_small(ha):
    features = ha.generate_synthetic(600, 12, "gaussian", seed=11)
    schema, attrs = ha.generate_attributes(600, 3, 3, seed=12)
    stats = ha.sample_statistics(features, attrs, 300, seed=13)
    config = ha.compute_alpha(stats, features.shape[0], schema.l)
    params = ha.BuildParams(gamma=24, gamma_new=24, seed=3)
    st, graph = staged_build(ha, features, attrs, schema, params, config)
    qf, qa, qm = ha.generate_queries(features, attrs, 20, 3, min_matches=5, seed=14)
    qm = qm.copy()
    qm[5:10, 1] = 0  # partial masks: a wildcard dimension on a third of the queries
    qm[10:13] = 0
    st.update(searches(ha, graph, qf, qa, [1, 2, 15, 30, 60], masks=qm))
    st.update({f"nomask_{k}": v for k, v in searches(ha, graph, qf, qa, [10], coarse=(True,)).items()})
    gt = np.stack([ha.oracle_auto_topk(features, attrs, qf[i], qa[i], 20, config, qm[i])
                   for i in range(qf.shape[0])])
    st.update(features=features, attrs=attrs, alpha=np.float64(config.alpha),
              s_v=np.float64(stats.avg_feature_distance), s_a=np.float64(stats.avg_attribute_distance),
              qf=qf, qa=qa, qm=qm, oracle_top20=gt, gamma=np.int64(24), sigma=np.float64(params.sigma))
    return st


def case_overflow(ha):
    rng = np.random.default_rng(5)
    n, d = 1500, 32
    features = rng.standard_normal((n, d), dtype=np.float32)
    attrs = rng.integers(1, 5, (n, 1), dtype=np.int32)
    schema = ha.AttributeSchema(dictionaries=(("a", "b", "c", "d"),))
    stats = ha.sample_statistics(features, attrs, 500, seed=0)
    config = ha.compute_alpha(stats, n, 1)
    params = ha.BuildParams(gamma=12, gamma_new=12, sigma=0.44, seed=9)
    st, graph = staged_build(ha, features, attrs, schema, params, config)
    qf = rng.standard_normal((30, d), dtype=np.float32)
    qa = rng.integers(1, 5, (30, 1), dtype=np.int32)
    st.update(searches(ha, graph, qf, qa, [5, 12]))
    st.update(features=features, attrs=attrs, alpha=np.float64(config.alpha), qf=qf, qa=qa,
              gamma=np.int64(12), sigma=np.float64(params.sigma))
    return st


def cfg1_data():
    rng = np.random.default_rng(0)
    X = rng.standard_normal((10000, 32), dtype=np.float32)
    A = rng.integers(1, 5, (10000, 1), dtype=np.int32)
    QX = rng.standard_normal((200, 32), dtype=np.float32)
    QA = rng.integers(1, 5, (200, 1), dtype=np.int32)
    return X, A, QX, QA


def case_cfg1(ha):
    X, A, QX, QA = cfg1_data()
    schema = ha.AttributeSchema(dictionaries=(tuple(f"v{i}" for i in range(1, 5)),))
    stats = ha.sample_statistics(X, A, 1000, seed=0)
    config = ha.compute_alpha(stats, X.shape[0], 1)
    params = ha.BuildParams()
    t0 = time.time()
    st, graph = staged_build(ha, X, A, schema, params, config)
    print(f"cfg1 build {time.time() - t0:.1f}s psi={st['psi_history']}", flush=True)
    out = {"alpha": np.float64(config.alpha), "psi_history": st["psi_history"],
           "iterations": st["iterations"], "q_sample": st["q_sample"], "q_gt": st["q_gt"],
           "reconnect_sweeps": st["reconnect_sweeps"]}
    for key, val in st.items():
        if isinstance(val, np.ndarray) and val.ndim == 2:
            out[f"sha_{key}"] = np.array(sha(val))
    for key in ("prune_counts", "reinf_counts", "final_counts", "indeg0", "prune_indeg"):
        out[f"sha_{key}"] = np.array(sha(st[key]))
    out["edges"] = np.array([st["init_ids"].size, int(st["prune_counts"].sum()),
                             int(st["final_counts"].sum())], np.int64)
    # first 50 rows of every stage in full, for diagnosable diffs
    for key in ("init_ids", "init_dists", "it1_ids", "it1_dists", "it1_flags", "prune_ids",
                "prune_counts", "final_ids", "final_dists", "final_counts"):
        out[f"head_{key}"] = st[key][:50].copy()
    out.update(searches(ha, graph, QX, QA, [10, 25, 50], coarse=(True,)))
    out["oracle_top10"] = np.stack([ha.oracle_auto_topk(X, A, QX[i], QA[i], 10, config)
                                    for i in range(QX.shape[0])])
    return out


def case_rng(ha):
    from hybridann.graph import init_random_graph
    out = {}
    grid = [(1000, 1), (1000, 50), (1000, 1000), (10000, 10), (10000, 500), (10001, 10),
            (10001, 201), (10001, 5000), (100000, 25), (100000, 3000), (1000000, 10),
            (1000000, 1000), (1000000, 20001), (2000000, 100)]
    for n, k in grid:
        for seed, qi in ((0, 0), (0, 7), (3, 199), (12345, 2**31 + 5)):
            ep = ha.entry_points(n, k, seed, qi)
            if k > 1000:  # large draws pinned by hash + head to keep the fixture small
                out[f"epsha_{n}_{k}_{seed}_{qi}"] = np.array(sha(ep))
                out[f"ephead_{n}_{k}_{seed}_{qi}"] = ep[:256].copy()
            else:
                out[f"ep_{n}_{k}_{seed}_{qi}"] = ep
    # init ids before distances: gamma ids per node, shift, duplicate resample
    for n, g, seed in ((300, 24, 3), (5000, 100, 0), (20001, 64, 7)):
        rng = np.random.default_rng(seed)
        ids = rng.integers(0, n - 1, size=(n, g), dtype=np.int64)
        ids += ids >= np.arange(n)[:, None]
        srt = np.sort(ids, axis=1)
        bad = np.nonzero(np.any(srt[:, 1:] == srt[:, :-1], axis=1))[0]
        for i in bad:
            pool = np.concatenate((np.arange(i), np.arange(i + 1, n)))
            ids[i] = rng.choice(pool, size=g, replace=False)
        out[f"initsha_{n}_{g}_{seed}"] = np.array(sha(ids.astype(np.int32)))
        if n <= 5000:
            out[f"init_{n}_{g}_{seed}"] = ids.astype(np.int32)
        out[f"initbad_{n}_{g}_{seed}"] = bad.astype(np.int64)
    # the reference's own init (graph.py:120-129) agrees with the restatement above
    f = np.zeros((300, 2), np.float32)
    a = np.ones((300, 1), np.int32)
    schema = ha.AttributeSchema(dictionaries=(("x",),))
    g = init_random_graph(f, a, schema, ha.BuildParams(gamma=24, gamma_new=24, seed=3),
                          ha.MetricConfig.manual(1.0, 1))
    assert set(map(tuple, np.sort(g.nbr_ids, 1))) == set(map(tuple, np.sort(out["init_300_24_3"], 1)))
    return out


def case_index(ha):
    """The reference writes the small case's graph with its own write_index (graph.py:287-330)
    -> small_index.help (kept beside the .npz); its read_index of that file, searched at two
    pool sizes (ids, dists, stats), is pinned here."""
    features = ha.generate_synthetic(600, 12, "gaussian", seed=11)
    schema, attrs = ha.generate_attributes(600, 3, 3, seed=12)
    stats = ha.sample_statistics(features, attrs, 300, seed=13)
    config = ha.compute_alpha(stats, features.shape[0], schema.l)
    graph = ha.build(features, attrs, schema, ha.BuildParams(gamma=24, gamma_new=24, seed=3), config)
    path = os.path.join(OUT, "small_index.help")
    ha.write_index(graph, path)
    back = ha.read_index(path)
    qf, qa, _ = ha.generate_queries(features, attrs, 20, 3, min_matches=5, seed=14)
    out = searches(ha, back, qf, qa, [10, 30], coarse=(True,))
    # the reference's bench_sweep over the read-back graph (evaluate.py:95-141): recall and
    # distance evaluations are deterministic (QPS is not); and its CSV of fixed rows
    gt = [ha.oracle_auto_topk(features, attrs, qf[i], qa[i], 10, config) for i in range(qf.shape[0])]
    rows = ha.bench_sweep(back, qf, qa, gt, [5, 10, 30], timing_passes=1)
    out["sweep"] = np.array([[r.k, r.pioneer, r.mean_recall_at_10, r.mean_dist_evals, r.n_queries]
                             for r in rows], np.float64)
    out["sweep_gt"] = np.stack(gt)
    from hybridann.evaluate import SweepRow, write_sweep_csv
    fixed = [SweepRow(k=10, pioneer=5, mean_recall_at_10=0.95123456, qps=1234.5678,
                      mean_dist_evals=321.123, n_queries=20),
             SweepRow(k=200, pioneer=100, mean_recall_at_10=1.0, qps=7.0, mean_dist_evals=4152.84, n_queries=10000)]
    csv_path = os.path.join("/tmp", "ref_sweep.csv")
    write_sweep_csv(csv_path, fixed)
    out["sweep_csv"] = np.array(open(csv_path).read())
    out.update(qf=qf, qa=qa, counts=back.nbr_counts.copy(), ids=back.nbr_ids.copy(),
               dists=back.nbr_dists.copy(), file_sha=np.array(hashlib.sha256(open(path, "rb").read()).hexdigest()))
    return out


def main():
    sys.path.insert(0, REF)
    import hybridann as ha
    which = sys.argv[1:] or ["small", "overflow", "rng", "cfg1"]
    for name in which:
        t0 = time.time()
        data = globals()[f"case_{name}"](ha)
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **data)
        print(f"{name}: {len(data)} arrays, {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()

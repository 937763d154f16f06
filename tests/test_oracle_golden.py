"""Pin the CPU oracle (oracle/) against golden vectors produced by the reference.

These run on CPU (no GPU needed).  The oracle must reproduce the reference
bit for bit at every build stage and for every search, so that the GPU parity
tests can trust it as the checker.
"""

import hashlib

import numpy as np
import pytest

from oracle import oracle as O


def sha(a):
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes() + str(a.dtype).encode() + str(a.shape).encode()).hexdigest()


def _staged(gd, gamma, sigma, seed, psi_target=0.8):
    snaps, stages = [], {}
    g = O.run_descent(gd["features"], gd["attrs"], float(gd["alpha"]), gamma=gamma,
                      gamma_new=gamma, psi_target=psi_target, seed=seed, snapshots=snaps)
    O.semantic_prune(g, sigma, stages)
    return g, snaps, stages


def _check_stages(gd, g, snaps, stages):
    np.testing.assert_array_equal(snaps[0][0], gd["init_ids"])
    np.testing.assert_array_equal(snaps[0][1], gd["init_dists"])
    assert g.log["iterations"] == int(gd["iterations"])
    np.testing.assert_array_equal(np.array(g.log["psi_history"]), gd["psi_history"])
    np.testing.assert_array_equal(g.log["sample_ids"], gd["q_sample"])
    np.testing.assert_array_equal(g.log["gt"], gd["q_gt"])
    for it in range(1, g.log["iterations"] + 1):
        ids, dists, flags = snaps[it]
        np.testing.assert_array_equal(ids, gd[f"it{it}_ids"])
        np.testing.assert_array_equal(dists, gd[f"it{it}_dists"])
        np.testing.assert_array_equal(flags, gd[f"it{it}_flags"])
    for key in ("indeg0", "prune_ids", "prune_dists", "prune_counts", "prune_indeg",
                "reinf_ids", "reinf_dists", "reinf_counts"):
        np.testing.assert_array_equal(stages[key], gd[key], err_msg=key)
    assert g.log["reconnect_sweeps"] == int(gd["reconnect_sweeps"])
    np.testing.assert_array_equal(g.nbr_ids, gd["final_ids"])
    np.testing.assert_array_equal(g.nbr_dists, gd["final_dists"])
    np.testing.assert_array_equal(g.nbr_counts, gd["final_counts"])


def _check_searches(gd, g, qf, qa, masks=None, prefix="s_"):
    keys = sorted(k for k in gd.files if k.startswith(prefix) and k.endswith("_ids"))
    assert keys
    for key in keys:
        tag = key[len(prefix):-len("_ids")]
        k = int(tag.split("_")[0][1:])
        coarse = tag.endswith("_c")
        ids, dists, st = O.search_batch(g.features, g.attrs, g.nbr_ids, g.nbr_counts, g.alpha,
                                        qf, qa, k, masks=masks, use_coarse=coarse)
        np.testing.assert_array_equal(ids, gd[key], err_msg=key)
        np.testing.assert_array_equal(dists, gd[f"{prefix}{tag}_dists"], err_msg=key)
        np.testing.assert_array_equal(st, gd[f"{prefix}{tag}_stats"], err_msg=key)


def test_small_build_every_stage(small_golden):
    gd = small_golden
    g, snaps, stages = _staged(gd, 24, float(gd["sigma"]), 3)
    _check_stages(gd, g, snaps, stages)


def test_small_searches_and_oracle(small_golden):
    gd = small_golden
    g, _, _ = _staged(gd, 24, float(gd["sigma"]), 3)
    qm = gd["qm"].astype(np.float64)
    _check_searches(gd, g, gd["qf"], gd["qa"], masks=qm)
    _check_searches(gd, g, gd["qf"], gd["qa"], masks=None, prefix="nomask_s_")
    for qi in range(gd["qf"].shape[0]):
        got = O.oracle_auto_topk(gd["features"], gd["attrs"], gd["qf"][qi], gd["qa"][qi], 20,
                                 float(gd["alpha"]), gd["qm"][qi])
        np.testing.assert_array_equal(got, gd["oracle_top20"][qi])


def test_overflow_build_every_stage(overflow_golden):
    gd = overflow_golden
    g, snaps, stages = _staged(gd, 12, float(gd["sigma"]), 9)
    assert g.log["full_merges"] > 0, "case must exercise the reinforce overflow path"
    assert int(gd["reconnect_sweeps"]) >= 1
    _check_stages(gd, g, snaps, stages)
    _check_searches(gd, g, gd["qf"], gd["qa"])


def test_alpha_matches_reference(small_golden):
    gd = small_golden
    s_v, s_a = O.sample_statistics(gd["features"], gd["attrs"], 300, seed=13)
    assert s_v == float(gd["s_v"]) and s_a == float(gd["s_a"])
    assert O.compute_alpha(s_v, s_a, 600, 3) == float(gd["alpha"])


def test_alpha_published_known_answer():
    # reference test_metric.py:66-71 — SIFT statistics, N=1M, L=3 give alpha = 0.743
    a = O.compute_alpha(536.93, 1.67, 1_000_000, 3)
    assert a == pytest.approx(0.743, abs=1e-3)


def test_np_row_sum_matches_numpy():
    rng = np.random.default_rng(0)
    for m in (1, 3, 7, 8, 9, 12, 16, 31, 32, 33, 96, 100, 127, 128, 129, 200, 960):
        a = rng.standard_normal((50, m)) ** 2
        want = a.sum(axis=1)
        got = np.array([O.lib().or_np_row_sum(np.ascontiguousarray(r), m) for r in a])
        np.testing.assert_array_equal(got, want, err_msg=f"m={m}")


def test_oracle_tie_break_by_id():
    # reference test_evaluate.py:24-29
    f = np.zeros((5, 2), np.float32)
    a = np.ones((5, 1), np.int32)
    got = O.oracle_auto_topk(f, a, np.ones(2, np.float32), np.array([1]), 5, 1.0)
    np.testing.assert_array_equal(got, [0, 1, 2, 3, 4])


@pytest.mark.slow
def test_cfg1_goldens(cfg1_golden):
    """BASELINE config 1 end to end: psi history, edges, stage hashes, searches, GT."""
    gd = cfg1_golden
    rng = np.random.default_rng(0)
    X = rng.standard_normal((10000, 32), dtype=np.float32)
    A = rng.integers(1, 5, (10000, 1), dtype=np.int32)
    QX = rng.standard_normal((200, 32), dtype=np.float32)
    QA = rng.integers(1, 5, (200, 1), dtype=np.int32)
    s_v, s_a = O.sample_statistics(X, A, 1000, seed=0)
    alpha = O.compute_alpha(s_v, s_a, 10000, 1)
    assert alpha == float(gd["alpha"])
    snaps, stages = [], {}
    g = O.run_descent(X, A, alpha, snapshots=snaps)
    O.semantic_prune(g, 0.44, stages)
    np.testing.assert_array_equal(np.array(g.log["psi_history"]), gd["psi_history"])
    assert sha(snaps[0][0]) == str(gd["sha_init_ids"])
    assert sha(snaps[0][1]) == str(gd["sha_init_dists"])
    for it in range(1, int(gd["iterations"]) + 1):
        assert sha(snaps[it][0]) == str(gd[f"sha_it{it}_ids"])
        assert sha(snaps[it][1]) == str(gd[f"sha_it{it}_dists"])
        assert sha(snaps[it][2]) == str(gd[f"sha_it{it}_flags"])
    assert sha(stages["prune_ids"]) == str(gd["sha_prune_ids"])
    assert sha(stages["prune_counts"]) == str(gd["sha_prune_counts"])
    assert sha(g.nbr_ids) == str(gd["sha_final_ids"])
    assert sha(g.nbr_dists) == str(gd["sha_final_dists"])
    assert sha(g.nbr_counts) == str(gd["sha_final_counts"])
    np.testing.assert_array_equal(gd["edges"], [1_000_000, 130_250, 194_468])
    for k in (10, 25, 50):
        ids, dists, st = O.search_batch(X, A, g.nbr_ids, g.nbr_counts, alpha, QX, QA, k, nthreads=0)
        np.testing.assert_array_equal(ids, gd[f"s_k{k}_c_ids"])
        np.testing.assert_array_equal(dists, gd[f"s_k{k}_c_dists"])
        np.testing.assert_array_equal(st, gd[f"s_k{k}_c_stats"])
    # SURVEY §4 goldens: K=50 totals over 200 queries
    np.testing.assert_array_equal(gd["s_k50_c_stats"].sum(0), [185910, 61861, 5397, 10014])
    for qi in range(0, 200, 7):
        np.testing.assert_array_equal(O.oracle_auto_topk(X, A, QX[qi], QA[qi], 10, alpha),
                                      gd["oracle_top10"][qi])


# ---- the parallel restatement (stable_oracle.c or_*_x, oracle.ParallelKernels) ---------------

def _staged_par(gd, gamma, sigma, seed, nthreads, psi_target=0.8):
    snaps, stages = [], {}
    g = O.run_descent(gd["features"], gd["attrs"], float(gd["alpha"]), gamma=gamma,
                      gamma_new=gamma, psi_target=psi_target, seed=seed, snapshots=snaps,
                      nthreads=nthreads)
    O.semantic_prune(g, sigma, stages, nthreads=nthreads)
    return g, snaps, stages


@pytest.mark.parametrize("nthreads", [0, 3])
def test_parallel_build_small_every_stage(small_golden, nthreads):
    gd = small_golden
    g, snaps, stages = _staged_par(gd, 24, float(gd["sigma"]), 3, nthreads)
    _check_stages(gd, g, snaps, stages)


@pytest.mark.parametrize("nthreads", [0, 2])
def test_parallel_build_overflow_every_stage(overflow_golden, nthreads):
    gd = overflow_golden
    g, snaps, stages = _staged_par(gd, 12, float(gd["sigma"]), 9, nthreads)
    assert g.log["full_merges"] > 0
    _check_stages(gd, g, snaps, stages)


def _u8_or_real(kind, n, m, l, card, rng):
    if kind == "u8":
        centres = rng.uniform(0, 255, (20, m))
        x = np.clip(np.rint(centres[rng.integers(0, 20, n)] + 25 * rng.standard_normal((n, m))), 0, 255)
    elif kind == "dup":  # exact duplicate rows: zero-length offsets, cosine 1.0, ties by id
        base = rng.integers(0, 4, (n // 3, m))
        x = base[rng.integers(0, n // 3, n)]
    else:
        x = rng.standard_normal((n, m)) * np.exp(rng.uniform(-1, 1, m))
    return x.astype(np.float32), rng.integers(1, card + 1, (n, l)).astype(np.int32)


@pytest.mark.parametrize("kind,n,m,l,card,gamma,sigma", [
    ("u8", 3000, 64, 2, 3, 24, 0.44), ("real", 3000, 37, 1, 5, 20, 0.3),
    ("real", 2500, 13, 2, 2, 32, 0.6), ("dup", 1500, 8, 1, 2, 16, 0.44),
    ("u8", 1200, 128, 3, 2, 40, 0.2)])
def test_parallel_build_equals_sequential(kind, n, m, l, card, gamma, sigma):
    """Every stage of the parallel build against the reference's loops on data the goldens do
    not cover: exact u8 sums, d % 4 != 0 (the 4-lane fp64 tail), duplicates, heavy pruning."""
    rng = np.random.default_rng(n + m)
    X, A = _u8_or_real(kind, n, m, l, card, rng)
    s_v, s_a = O.sample_statistics(X, A, min(500, n), seed=0)
    alpha = O.compute_alpha(s_v, s_a, n, l)
    seq_s, seq_st, par_s, par_st = [], {}, [], {}
    g1 = O.run_descent(X, A, alpha, gamma=gamma, gamma_new=gamma, snapshots=seq_s, nthreads=1)
    g2 = O.run_descent(X, A, alpha, gamma=gamma, gamma_new=gamma, snapshots=par_s, nthreads=0)
    assert g1.log["psi_history"] == g2.log["psi_history"]
    assert g1.log["pairs"] == g2.log["pairs"]
    for a, b in zip(seq_s, par_s):
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)
    O.semantic_prune(g1, sigma, seq_st, nthreads=1)
    O.semantic_prune(g2, sigma, par_st, nthreads=0)
    for key in seq_st:
        np.testing.assert_array_equal(seq_st[key], par_st[key], err_msg=key)
    np.testing.assert_array_equal(g1.nbr_counts, g2.nbr_counts)
    np.testing.assert_array_equal(g1.nbr_ids, g2.nbr_ids)
    np.testing.assert_array_equal(g1.nbr_dists, g2.nbr_dists)
    assert g1.log["full_merges"] == g2.log["full_merges"]


def test_u8_copy_only_for_exact_bytes():
    assert O.u8_copy(np.array([[0, 255.0]], np.float32)) is not None
    assert O.u8_copy(np.array([[0, 256.0]], np.float32)) is None
    assert O.u8_copy(np.array([[-1, 2.0]], np.float32)) is None
    assert O.u8_copy(np.array([[0.5, 2.0]], np.float32)) is None


def test_hybrid_groundtruth_restatement():
    # reference test_evaluate.py:40-49: exact-match filter, fewer than k when matches are scarce
    f = np.array([[0, 0], [1, 0], [2, 0], [3, 0]], np.float32)
    a = np.array([[1, 1], [1, 2], [1, 1], [2, 1]], np.int32)
    np.testing.assert_array_equal(O.oracle_hybrid_groundtruth(f, a, [0, 0], [1, 1], 5), [0, 2])
    np.testing.assert_array_equal(O.oracle_hybrid_groundtruth(f, a, [0, 0], [1, 1], 5, mask=[1, 0]),
                                  [0, 1, 2])
    assert O.oracle_hybrid_groundtruth(f, a, [0, 0], [9, 9], 5).size == 0

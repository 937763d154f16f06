"""Small end-to-end run of every device path for compute-sanitizer (memcheck / racecheck /
synccheck): HELP build + routed search + exact top-k on real-valued data (fp64 rows, TF32
filter), on integer data in [0, 255] (u8 / dp4a routing, tcgen05 kind::i8 top-k, u8 prune),
with the reinforce overflow replay, reconnect sweep, k > 32 two-pass top-k, large-K routing
and the exact-match ground truth.  python tools/sanitize_run.py [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2604_01617_b200 as sb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
rng = np.random.default_rng(0)
for kind in ("real", "u8"):
    if kind == "real":
        X = rng.standard_normal((n, 32)).astype(np.float32)
        QX = rng.standard_normal((40, 32))
    else:
        X = np.clip(np.rint(rng.normal(128, 40, (n, 32))), 0, 255).astype(np.float32)
        QX = np.clip(np.rint(rng.normal(128, 40, (40, 32))), 0, 255)
    A = rng.integers(1, 4, (n, 2)).astype(np.int32)
    QA = rng.integers(1, 4, (40, 2))
    cfg = sb.compute_alpha(sb.sample_statistics(X, A, 500, seed=0), n, 2)
    # small gamma with a high sigma: reinforce overflows and a reconnect sweep runs
    g = sb.build(X, A, sb.AttributeSchema((("a", "b", "c"),) * 2),
                 sb.BuildParams(gamma=12, gamma_new=12, sigma=0.9, seed=1), cfg)
    for k in (10, 40):
        sb.search_batch_arrays(g, QX, QA, sb.SearchParams(k=k))
    sb.search_batch_arrays(g, QX[:4], QA[:4], sb.SearchParams(k=min(n, 1500)))
    for k in (10, 64):
        sb.oracle_auto_topk_batch(X, A, QX, QA, k, cfg)
    sb.evaluate.oracle_hybrid_groundtruth_batch(X, A, QX, QA, 10)
    print(kind, "ok", g.build_log.get("reinforce_overflow_rows"), g.build_log.get("reconnect_sweeps"), flush=True)

"""Full-scale parity of the B200 path against the CPU oracle at every BASELINE config.

For each config recipe (tools/configs.py) at its full N: the GPU HELP build and the oracle's
build (parallel restatement of the reference's loops on all host cores, pinned bit-exact to
the reference in tests/test_oracle_golden.py and tests/test_ref_swap.py) must give the same
graph bit for bit; the GPU exact AUTO top-k must equal the oracle's on a 100-query sample;
GPU routing must equal the oracle's (ids, fp64 distances, SearchStats) on a query sample at
the config's operating K.  One JSON line per config (build seconds on both sides included).

  python tools/parity_full.py [--configs cfg2,cfg3,...] [--out profiles/parity_full_r2.jsonl]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# operating pool sizes K* measured in round 1 (profiles/configs_r1.jsonl), route sample size
OPERATING = {"cfg2": (200, 500), "cfg3": (6000, 40), "cfg4": (500, 200), "cfg5c1": (500, 200),
             "cfg5c10": (200, 500), "cfg5c100": (500, 200), "cfg5c1000": (4000, 40),
             "cfg5c10000": (32000, 8)}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run(cfg: str) -> dict:
    import paper_2604_01617_b200 as sb
    from oracle import oracle as O
    from tools.configs import make_config
    t0 = time.perf_counter()
    X, A, QX, QA, card = make_config(cfg)
    gen_s = time.perf_counter() - t0
    n = X.shape[0]
    m = sb.compute_alpha(sb.sample_statistics(X, A, min(1000, n), seed=0), n, A.shape[1])
    schema = sb.AttributeSchema(tuple(tuple(str(i) for i in range(c)) for c in card))
    t0 = time.perf_counter()
    g = sb.build(X, A, schema, sb.BuildParams(), m)
    gpu_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    og = O.build(X, A, m.alpha, sigma=0.44, gamma=100, gamma_new=100, nthreads=0)
    cpu_s = time.perf_counter() - t0
    mask = np.arange(g.nbr_ids.shape[1])[None, :] < og.nbr_counts[:, None]
    graph_equal = bool(np.array_equal(g.nbr_counts, og.nbr_counts) and
                       np.array_equal(np.where(mask, g.nbr_ids, -1), np.where(mask, og.nbr_ids, -1)) and
                       np.array_equal(np.where(mask, g.nbr_dists, 0), np.where(mask, og.nbr_dists, 0)))
    out = {"config": cfg, "n": n, "d": X.shape[1], "cards": list(card), "gen_s": round(gen_s, 2),
           "gpu_build_s": round(gpu_s, 3), "cpu_build_s": round(cpu_s, 2),
           "cpu_threads": os.cpu_count(), "cpu_model": cpu_model(),
           "graph_equal": graph_equal, "edges": int(og.nbr_counts.sum()),
           "psi_history_equal": g.build_log["psi_history"] == og.log["psi_history"],
           "pairs_equal": g.build_log["pairs"] == og.log["pairs"],
           "pairs": og.log["pairs"], "iterations": og.log["iterations"],
           "overflow_rows_gpu": int(g.build_log.get("reinforce_overflow_rows", 0)),
           "full_merges_cpu": int(og.log["full_merges"]),
           "reconnect_sweeps": int(og.log["reconnect_sweeps"])}
    # exact ground truth on a 100-query sample (k = 10, and k = 100 for cfg 3)
    for k in ((10, 100) if cfg == "cfg3" else (10,)):
        s = 100
        t0 = time.perf_counter()
        gi, gd = sb.oracle_auto_topk_batch(X, A, QX[:s], QA[:s], k, m, return_dists=True)
        ok = True
        for i in range(s):
            wi, wd = O.oracle_auto_topk(X, A, QX[i], QA[i], k, m.alpha, return_dists=True)
            ok = ok and np.array_equal(gi[i], wi) and np.array_equal(gd[i], wd)
        out[f"gt_k{k}_equal_on_{s}"] = bool(ok)
        out[f"gt_k{k}_check_s"] = round(time.perf_counter() - t0, 2)
    K, q = OPERATING.get(cfg, (100, 100))
    K = min(K, n)
    t0 = time.perf_counter()
    got = sb.search_batch_arrays(g, QX[:q], QA[:q], sb.SearchParams(k=K))
    want = O.search_batch(X, A, og.nbr_ids, og.nbr_counts, m.alpha, QX[:q], QA[:q], K, nthreads=0)
    out.update({"route_K": K, "route_queries": q,
                "route_equal": bool(np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
                                    and np.array_equal(got[2][:, :4], want[2])),
                "route_check_s": round(time.perf_counter() - t0, 2)})
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--configs", default="cfg2,cfg3,cfg4,cfg5c1,cfg5c10,cfg5c100,cfg5c1000,cfg5c10000")
    p.add_argument("--out", default=os.path.join(ROOT, "profiles", "parity_full_r2.jsonl"))
    a = p.parse_args()
    for cfg in a.configs.split(","):
        r = run(cfg)
        print(json.dumps(r), flush=True)
        with open(a.out, "a") as f:
            f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()

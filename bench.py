#!/usr/bin/env python
"""bench.py — hybrid QPS @ Recall@10 >= 0.95 on one B200, HELP build seconds, and routing HBM
GB/s vs the measured peak, on BASELINE.json configs[1] (cfg 2: N=1M, d=128 integer-valued
clustered features, 3 attributes 3/5/10, 10,000 queries with a full constraint, k=10).

One step = one pass of the hot path over one batch: search_batch of all queries at the
operating pool size K* (the smallest K of the sweep whose mean Recall@10 against the exact
AUTO ground truth is >= 0.95).  Data are seeded synthetic stand-ins (tools/configs.py).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mine|reference] [--config cfg2]

N > 1 (torchrun, one rank per GPU): every rank holds a replica of the index and the 10k-query
batch is split across the ranks (sharding.search_batch_sharded_device: each rank routes its
block, one NCCL all-gather per output assembles the results on every GPU) — strong scaling,
max-over-ranks device time.  The node-sharded exact ground truth (one all-gather exchange) is
timed beside it.

--impl reference times the reference's CPU implementation of the path (the oracle port in
oracle/; the reference is Python + Numba with no native code to build) on all host cores:
it builds the HELP index of the same data on the CPU (timed: the CPU "HELP build s"), then
routes bounded samples of the same queries at the same K*.  It never loads the B200 library.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "hybrid QPS @ recall@10>=0.95 (1 B200); HELP build s; HBM GB/s vs peak"
UNIT = "queries/s"
K_SWEEP = [10, 20, 25, 30, 50, 100, 200, 300, 500, 750, 1000, 1500, 2000, 3000, 4000]
GAMMA = 100  # BuildParams defaults (graph.py:26-33)


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["mine", "reference"], default="mine")
    p.add_argument("--config", default="cfg2")
    p.add_argument("--n", type=int, default=None, help="override N (testing only)")
    p.add_argument("--kcap", type=int, default=4000)
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--no-topk", action="store_true",
                   help="skip the exhaustive top-k tensor-core rooflines")
    p.add_argument("--no-legs", action="store_true",
                   help="skip the real-valued routing legs (cfg 4, cfg 5 cardinality 10)")
    p.add_argument("--no-cpu-build", action="store_true",
                   help="skip the CPU oracle build + graph parity of the mine arm")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        rows = []
        for r in csv.reader(io.StringIO(open(self.path).read())):
            r = [x.strip() for x in r]
            if len(r) >= 9:
                rows.append(r)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def measured_hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        v = float(json.load(open(path))["hbm_gbs"])
        return v, "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(config_name):
    """dram bytes per route_kernel launch from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", f"route_ncu_{config_name}.json")
    try:
        d = json.load(open(path))
        return float(d["dram_bytes_per_launch"])
    except Exception:
        return None


# ---------------------------------------------------------------------------------------
def load_workload(args):
    from tools.configs import make_config
    return make_config(args.config, args.n)


def bench_config(args, n, m, l, card, q, kstar, pioneer, features_bytes):
    """The workload description both arms print (identical dicts: same config)."""
    return {
        "workload": f"{args.config}: N={n:,} d={m} L={l} cards={list(card)} Q={q} k=10",
        "operating_K": int(kstar), "pioneer": int(pioneer),
        "index": "HELP gamma=100 gamma_new=100 sigma=0.44 psi_target=0.8 (BuildParams defaults)",
        "l2": "inputs larger than L2 (features %.0f MB + adjacency %.0f MB vs 126 MB L2)"
              % (features_bytes / 1e6, n * GAMMA * 8 / 1e6),
    }


def build_index(X, A, card):
    import paper_2604_01617_b200 as sb
    cfg = sb.compute_alpha(sb.sample_statistics(X, A, min(1000, X.shape[0]), seed=0),
                           X.shape[0], A.shape[1])
    schema = sb.AttributeSchema(tuple(tuple(str(i) for i in range(c)) for c in card))
    t0 = time.perf_counter()
    g = sb.build(X, A, schema, sb.BuildParams(), cfg)
    return g, cfg, time.perf_counter() - t0


def sweep_operating_point(g, cfg, X, A, QX, QA, kcap):
    import paper_2604_01617_b200 as sb
    t0 = time.perf_counter()
    gt = sb.oracle_auto_topk_batch(X, A, QX, QA, 10, cfg)
    gt_s = time.perf_counter() - t0
    table = []
    kstar = None
    for k in K_SWEEP:
        if k > min(kcap, X.shape[0]):
            break
        ids, _, st = sb.search_batch_arrays(g, QX, QA, sb.SearchParams(k=k))
        rec = sb.mean_recall(ids, gt, 10)
        table.append({"k": k, "recall_at_10": round(rec, 6), "mean_dist_evals": float(st[:, 0].mean())})
        if rec >= 0.95:
            kstar = k
            break
    if kstar is None:
        kstar = table[-1]["k"]
    return kstar, table, gt, gt_s


def algorithmic_bytes(st, m, l, row_bytes=None, norm_bytes=0):
    """Routing bytes per SURVEY §8(d): evals*(row + 4L) + 4*(expansions + scanned), with the
    row as the kernel reads it (4d fp32, or d bytes + a 4-byte norm on the u8 path)."""
    rb = 4 * m if row_bytes is None else row_bytes
    evals = st[:, 0].astype(np.float64)
    exps = (st[:, 2] + st[:, 3]).astype(np.float64)
    scanned = st[:, 4].astype(np.float64)
    return float((evals * (rb + norm_bytes + 4 * l) + 4 * (exps + scanned)).sum())


def build_summary(g, build_s, n, m, l, cpu=None):
    """HELP build: seconds, distance evaluations (n*gamma init + join pairs +
    the psi ground truth's sample*n) per second, and the local join against the HBM roofline
    by §8(d)'s gather figure n*(gamma_new+gamma)*(4d+4L) bytes per descent iteration."""
    log = g.build_log
    pairs = [int(p) for p in log.get("pairs", [])]
    sample = 100 if n > 100 else n
    evals = n * GAMMA + sum(pairs) + sample * n
    t_iter = float(sum(log.get("seconds_iterations", [])))
    gath = len(pairs) * n * (2 * GAMMA) * (4 * m + 4 * l)
    peak, src = measured_hbm_peak()
    out = {"gpu_s": round(build_s, 3), "iterations": log.get("iterations"),
           "psi_history": log.get("psi_history"), "termination": log.get("termination"),
           "pairs": pairs, "dist_evals": int(evals),
           "gpu_dist_evals_per_s": round(evals / build_s, 1),
           "seconds_init": round(log.get("seconds_init", 0.0), 4),
           "seconds_iterations": [round(x, 4) for x in log.get("seconds_iterations", [])],
           "seconds_prune": round(log.get("seconds_prune", 0.0), 4),
           "prune_guard_rounds": log.get("prune_guard_rounds"),
           "reinforce_overflow_rows": log.get("reinforce_overflow_rows"),
           "join_roofline": {"bound": "hbm", "unit": "GB/s",
                             "achieved": round(gath / t_iter / 1e9, 1) if t_iter else None,
                             "peak": peak, "frac": round(gath / t_iter / 1e9 / peak, 4) if t_iter else None,
                             "bytes_def": "SURVEY 8(d): n*(gamma_new+gamma)*(4d+4L) per descent iteration",
                             "seconds": round(t_iter, 4), "peak_source": src,
                             "join_pairs_per_s": round(sum(pairs) / t_iter, 1) if t_iter else None}}
    if cpu:
        out.update(cpu)
        out["cpu_dist_evals_per_s"] = round(evals / cpu["cpu_s"], 1)
        out["speedup_vs_cpu"] = round(cpu["cpu_s"] / build_s, 1)
    return out


# ---------------------------------------------------------------------------------------
def run_mine(args, rank, world, local):
    import torch
    import paper_2604_01617_b200 as sb
    from paper_2604_01617_b200 import sharding
    from paper_2604_01617_b200.device import entry_points_host

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    X, A, QX, QA, card = load_workload(args)
    n, m = X.shape
    l = A.shape[1]
    q = QX.shape[0]
    g, cfg, build_s = build_index(X, A, card)
    kstar, table, gt, gt_s = sweep_operating_point(g, cfg, X, A, QX, QA, args.kcap)
    params = sb.SearchParams(k=kstar)
    P = params.resolved_pioneer_size()
    inv_alpha = 1.0 / cfg.alpha
    dev = g.device()
    # a dedicated (non-default) stream: kernels and CUDA events must share it
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    dev.set_stream(stream.cuda_stream)

    # ---- value: inputs resident in HBM, one device call per step ------------------------
    qf_d = torch.from_numpy(np.ascontiguousarray(QX, np.float64)).cuda()
    qa_d = torch.from_numpy(np.ascontiguousarray(QA, np.float64)).cuda()
    ids_d = torch.empty((q, kstar), dtype=torch.int64, device="cuda")
    dists_d = torch.empty((q, kstar), dtype=torch.float64, device="cuda")
    st_d = torch.empty((q, 5), dtype=torch.int64, device="cuda")

    def step_full(entries_ptr=None):
        dev.route_dev(qf_d.data_ptr(), qa_d.data_ptr(), None, q, kstar, P, inv_alpha,
                      ids_d.data_ptr(), dists_d.data_ptr(), st_d.data_ptr(),
                      entries_ptr=entries_ptr, seed=0, qi0=0)

    def step():
        if world == 1:
            step_full()
            return ids_d
        return sharding.search_batch_sharded_device(dev, qf_d, qa_d, q, kstar, P, inv_alpha)[0]

    for _ in range(max(3, args.warmup)):
        out_ids = step()
    torch.cuda.synchronize()
    # parity of the device path (sharded at N > 1) with the public API at K*
    ids_api, _, st_api = sb.search_batch_arrays(g, QX, QA, params)
    dev.set_stream(stream.cuda_stream)
    assert np.array_equal(out_ids.cpu().numpy(), ids_api), "device path != public API"
    gpu_index = int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local)).split(",")[local]) \
        if os.environ.get("CUDA_VISIBLE_DEVICES") else local
    sampler = ClockSampler(gpu_index)
    l0 = dev.launch_count()
    barrier()
    torch.cuda.synchronize()
    sampler.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    launches = dev.launch_count() - l0
    ms = e0.elapsed_time(e1) / args.steps
    ms = max_over_ranks(ms)
    value = q / (ms / 1000.0)  # the whole batch per step, split over the ranks

    # ---- roofline: the routing kernel alone over the full batch (entries precomputed) ----
    ent = entry_points_host(n, kstar, 0, 0, q)
    ent_d = torch.from_numpy(ent).cuda()
    step_full(ent_d.data_ptr())
    torch.cuda.synchronize()
    reps = max(3, min(args.steps, 10))
    r0 = torch.cuda.Event(enable_timing=True)
    r1 = torch.cuda.Event(enable_timing=True)
    r0.record(stream)
    for _ in range(reps):
        step_full(ent_d.data_ptr())
    r1.record(stream)
    torch.cuda.synchronize()
    route_ms = r0.elapsed_time(r1) / reps
    st = st_d.cpu().numpy()
    rinfo = dev.route_info()
    # §8(d)'s per-evaluation figure counts the fp32 row (4d + 4L); on integer data in [0, 255]
    # the kernel reads a d-byte u8 row plus a 4-byte norm instead, reported beside it
    abytes = algorithmic_bytes(st, m, l)
    read_bytes = algorithmic_bytes(st, m, l, rinfo["row_bytes"], 4 if rinfo["path"] == "u8-dp4a" else 0)
    achieved = abytes / (route_ms / 1000.0) / 1e9
    peak, peak_src = measured_hbm_peak()
    traffic = ncu_traffic(args.config)

    # ---- e2e: public API, host buffers (pinned), copies inside the timed region -----------
    qf_h = torch.empty((q, m), dtype=torch.float64, pin_memory=True).numpy()
    qa_h = torch.empty((q, l), dtype=torch.float64, pin_memory=True).numpy()
    qf_h[:] = QX
    qa_h[:] = QA
    dev.set_stream(None)

    def e2e_call():
        if world == 1:
            return sb.search_batch_arrays(g, qf_h, qa_h, params)
        return sharding.search_batch_sharded(g, qf_h, qa_h, params)

    # warm-up: two live result sets, so the page-locked result pool holds the two sets the
    # timed loop alternates between (no allocation inside the timed region)
    warm = [e2e_call() for _ in range(2)]
    del warm
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ids_h, dists_h, st_h = e2e_call()
    e2e_s = (time.perf_counter() - t0) / args.steps
    e2e_s = max_over_ranks(e2e_s)
    e2e = q / e2e_s
    h2d = qf_h.nbytes + qa_h.nbytes
    d2h = ids_h.nbytes + dists_h.nbytes + st_h.nbytes

    # ---- N > 1: the node-sharded exact ground truth (one all-gather exchange) -------------
    sharded_gt = None
    if world > 1:
        sharding.oracle_auto_topk_sharded(X, A, QX[:256], QA[:256], 10, cfg)  # warm
        barrier()
        t0 = time.perf_counter()
        si, _ = sharding.oracle_auto_topk_sharded(X, A, QX, QA, 10, cfg)
        gs = max_over_ranks(time.perf_counter() - t0)
        sharded_gt = {"seconds": round(gs, 4), "queries": q, "k": 10,
                      "equal_to_single_gpu": bool(np.array_equal(si, gt))}

    cpu = None
    topk = None
    legs = None
    cpu_build = None
    parity = None
    if rank == 0 and world == 1:
        # CPU baseline: the oracle port, one thread (the reference's search is single-threaded,
        # SPEC.md:466), bounded sample of the same queries
        cpu = cpu_baseline(g, cfg, QX, QA, kstar, args.cpu_seconds, ids_api)
        if not args.no_cpu_build:
            cpu_build, parity = cpu_build_and_parity(g, cfg, X, A, QX, QA, gt)
        if not args.no_topk:
            topk, legs = topk_and_legs(g, cfg, QX, QA, legs=not args.no_legs)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator with the config's shapes; tools/configs.py)",
            "config": bench_config(args, n, m, l, card, q, kstar, P, X.nbytes),
            "parallelism": "queries split over %d replicas, NCCL all-gather of results" % world
                           if world > 1 else "single GPU",
            "recall_at_10": table[-1]["recall_at_10"],
            "build_s": round(build_s, 3),
            "build": build_summary(g, build_s, n, m, l, cpu_build),
            "edges": int(g.nbr_counts.sum()),
            "gt_s": round(gt_s, 3),
            "sweep": table,
            "mean_dist_evals": float(st[:, 0].mean()),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": traffic, "kernel": "route_kernel",
                         "distance_path": rinfo["path"], "row_bytes": rinfo["row_bytes"],
                         "algorithmic_bytes_def": "SURVEY 8(d): dist_evals*(4d+4L) + 4*(expansions+scanned)",
                         "bytes_read_per_launch": read_bytes,
                         "frac_of_bytes_read": round(read_bytes / (route_ms / 1000.0) / 1e9 / peak, 4),
                         "kernel_ms": round(route_ms, 4),
                         "algorithmic_bytes_per_launch": abytes, "peak_source": peak_src,
                         "share_of_step": round(route_ms / ms, 3) if world == 1 else None},
            "e2e": {"value": round(e2e, 1), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches),
            "clocks": clocks,
            "cpu_baseline": cpu,
            "parity": parity,
            "sharded_ground_truth": sharded_gt,
            "roofline_topk": topk,
            "routing_legs": legs,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def cpu_build_and_parity(g, cfg, X, A, QX, QA, gt):
    """The CPU oracle (parallel restatement of the reference's loops, all host cores) builds
    the same index; its graph must equal the GPU's bit for bit.  The exact ground truth is
    cross-checked on a 100-query sample."""
    from oracle import oracle as O
    t0 = time.perf_counter()
    og = O.build(X, A, cfg.alpha, sigma=0.44, gamma=GAMMA, gamma_new=GAMMA, nthreads=0)
    cpu_s = time.perf_counter() - t0
    mask = np.arange(g.nbr_ids.shape[1])[None, :] < og.nbr_counts[:, None]
    equal = bool(np.array_equal(g.nbr_counts, og.nbr_counts) and
                 np.array_equal(np.where(mask, g.nbr_ids, -1), np.where(mask, og.nbr_ids, -1)) and
                 np.array_equal(np.where(mask, g.nbr_dists, 0), np.where(mask, og.nbr_dists, 0)))
    s = min(100, QX.shape[0])
    t0 = time.perf_counter()
    gt_ok = all(np.array_equal(O.oracle_auto_topk(X, A, QX[i], QA[i], 10, cfg.alpha), gt[i])
                for i in range(s))
    build = {"cpu_s": round(cpu_s, 2), "cpu_threads": os.cpu_count(), "cpu_model": cpu_model(),
             "cpu_kind": "port (oracle/stable_oracle.c parallel restatement, exact)",
             "graph_equal_to_cpu": equal}
    parity = {"graph_equal_to_cpu_oracle": equal, "edges_cpu": int(og.nbr_counts.sum()),
              "gt_parity_on_sample": bool(gt_ok), "gt_sample_queries": s,
              "gt_check_s": round(time.perf_counter() - t0, 2)}
    return build, parity


def peak_int8_tops():
    """Dense INT8 tensor throughput measured here: torch._int_mm 8192^3 (cuBLASLt, s8 x s8 ->
    s32), best of 10 (2 N^3 ops)."""
    import torch
    n = 8192
    a = torch.randint(-64, 64, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-64, 64, (n, n), dtype=torch.int8, device="cuda")
    for _ in range(3):
        torch._int_mm(a, b)
    best = 1e30
    for _ in range(10):
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        torch._int_mm(a, b)
        s1.record()
        s1.synchronize()
        best = min(best, s0.elapsed_time(s1) / 1e3)
    del a, b
    return 2 * n ** 3 / best / 1e12


def peak_tf32_tflops():
    """Dense TF32 tensor throughput measured here: cuBLAS fp32 8192^3 with TF32 allowed, best
    of 10 (MEASURED_PEAKS.json holds bf16 only)."""
    import torch
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    n = 8192
    a = torch.randn(n, n, device="cuda")
    b = torch.randn(n, n, device="cuda")
    for _ in range(3):
        a @ b
    best = 1e30
    for _ in range(10):
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        a @ b
        s1.record()
        s1.synchronize()
        best = min(best, s0.elapsed_time(s1) / 1e3)
    torch.backends.cuda.matmul.allow_tf32 = old
    del a, b
    return 2 * n ** 3 / best / 1e12


def _topk_entry(dev, QX, QA, k, alpha, n, m, peak, unit, peak_src):
    dev.bf_topk_queries(QX, QA, k, alpha)
    best = (1e30, 0.0)
    for _ in range(3):
        t0 = time.perf_counter()
        dev.bf_topk_queries(QX, QA, k, alpha)
        call = time.perf_counter() - t0
        best = min(best, (dev.bf_info()["kernel_ms"], call))
    info = dev.bf_info()
    q = QX.shape[0]
    rate = 2.0 * q * n * m / (best[0] / 1e3) / 1e12
    return {"path": info["path"], "queries": q, "nodes": n, "d": m, "k": k,
            "kernel_ms": round(best[0], 4), "call_ms": round(best[1] * 1e3, 3),
            "candidates_per_query": round(info["candidates"] / q, 1),
            "fallback_queries": info["fallback_queries"],
            "achieved": round(rate, 1), "unit": unit, "peak": round(peak, 1),
            "frac": round(rate / peak, 4), "peak_source": peak_src}


def routing_leg(name, X, A, QX, QA, card, kcap=4000):
    """A real-valued routing leg on another BASELINE config: HELP build, exact
    ground truth, the K sweep to Recall@10 >= 0.95 through the public API, then the routing
    kernel alone at K* over the full query batch (device-resident inputs, CUDA events) against
    the HBM roofline by §8(d)'s bytes, and the public-API QPS (host arrays in and out)."""
    import torch
    import paper_2604_01617_b200 as sb
    from paper_2604_01617_b200.device import entry_points_host
    g, cfg, build_s = build_index(X, A, card)
    kstar, table, _, gt_s = sweep_operating_point(g, cfg, X, A, QX, QA, kcap)
    q, m = QX.shape
    l = A.shape[1]
    params = sb.SearchParams(k=kstar)
    t0 = time.perf_counter()
    sb.search_batch_arrays(g, QX, QA, params)
    api_s = time.perf_counter() - t0
    dev = g.device()
    stream = torch.cuda.Stream()
    dev.set_stream(stream.cuda_stream)
    qf_d = torch.from_numpy(np.ascontiguousarray(QX, np.float64)).cuda()
    qa_d = torch.from_numpy(np.ascontiguousarray(QA, np.float64)).cuda()
    ent_d = torch.from_numpy(entry_points_host(X.shape[0], kstar, 0, 0, q)).cuda()
    ids_d = torch.empty((q, kstar), dtype=torch.int64, device="cuda")
    dists_d = torch.empty((q, kstar), dtype=torch.float64, device="cuda")
    st_d = torch.empty((q, 5), dtype=torch.int64, device="cuda")

    def run():
        dev.route_dev(qf_d.data_ptr(), qa_d.data_ptr(), None, q, kstar, params.resolved_pioneer_size(),
                      1.0 / cfg.alpha, ids_d.data_ptr(), dists_d.data_ptr(), st_d.data_ptr(),
                      entries_ptr=ent_d.data_ptr())
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    e0.record(stream)
    for _ in range(reps):
        run()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    dev.set_stream(None)
    st = st_d.cpu().numpy()
    abytes = algorithmic_bytes(st, m, l)
    peak, src = measured_hbm_peak()
    log = g.build_log
    out = {"workload": f"{name}: N={X.shape[0]:,} d={m} L={l} cards={list(card)} Q={q} k=10",
           "operating_K": int(kstar), "recall_at_10": table[-1]["recall_at_10"],
           "distance_path": dev.route_info()["path"],
           "build_s": round(build_s, 3), "build_seconds_prune": round(log.get("seconds_prune", 0.0), 3),
           "build_iterations_s": [round(x, 3) for x in log.get("seconds_iterations", [])],
           "reinforce_overflow_rows": log.get("reinforce_overflow_rows"),
           "gt_s": round(gt_s, 3), "kernel_ms": round(ms, 3), "qps_kernel": round(q / ms * 1e3, 1),
           "qps_public_api": round(q / api_s, 1), "mean_dist_evals": float(st[:, 0].mean()),
           "roofline": {"bound": "hbm", "achieved": round(abytes / (ms / 1e3) / 1e9, 1), "peak": peak,
                        "unit": "GB/s", "frac": round(abytes / (ms / 1e3) / 1e9 / peak, 4),
                        "algorithmic_bytes_per_launch": abytes, "peak_source": src}}
    dev.close()  # free the leg's device index before the next leg
    g._device = None
    return out


def topk_and_legs(g, cfg, QX, QA, legs=True):
    """Exhaustive AUTO top-k (oracle_auto_topk, evaluate.py:32-55) on the tensor cores, each
    against the measured dense peak of its precision: this config's ground truth (cfg 2: u8
    operands, tcgen05 kind::i8, exact; INT8 peak), cfg 3 at k = 10 and k = 100 and cfg 4 (both
    from the tools/configs.py recipes) on the TF32 filter + exact re-rank (TF32 peak).
    achieved = 2 q n d useful ops / the tensor-core pass (CUDA events inside the C ABI).
    With `legs`, the real-valued routing legs of cfg 4 and cfg 5 (cardinality 10) on the same
    generated data (routing_leg)."""
    import paper_2604_01617_b200 as sb
    from paper_2604_01617_b200.device import DeviceIndex
    from tools.configs import make_config
    i8 = peak_int8_tops()
    tf = peak_tf32_tflops()
    i8_src = "measured here: torch._int_mm s8 8192^3 best of 10"
    tf_src = "measured here: cuBLAS TF32 8192^3 best of 10"
    out = {"peaks": {"int8_tops": round(i8, 1), "tf32_tflops": round(tf, 1)}}
    route_legs = {}
    dev = g.device()
    n, m = g.features.shape
    out["bench_config"] = _topk_entry(dev, QX, QA, 10, cfg.alpha, n, m, i8, "TOP/s", i8_src)
    for name, ks in (("cfg3", (10, 100)), ("cfg4", (10,)), ("cfg5c10", ())):
        if not ks and not legs:
            continue
        X, A, QXc, QAc, card = make_config(name)
        if ks:
            mc = sb.compute_alpha(sb.sample_statistics(X, A, 1000, seed=0), X.shape[0], A.shape[1])
            d = DeviceIndex(X, A, 2)
            for k in ks:
                out[f"{name}_k{k}"] = _topk_entry(d, QXc, QAc, k, mc.alpha, X.shape[0], X.shape[1],
                                                  tf, "TFLOP/s", tf_src)
            d.close()
        if legs and name in ("cfg4", "cfg5c10"):
            route_legs[name] = routing_leg(name, X, A, QXc, QAc, card)
        del X, A
    return out, route_legs


def cpu_baseline(g, cfg, QX, QA, kstar, seconds, ids_gpu):
    """The oracle port (C restatement of _kernels.route + NumPy entry points) on the host."""
    from oracle import oracle as O
    f, a = g.features, g.attrs

    def run(lo, hi, threads):
        t0 = time.perf_counter()
        ids, _, _ = O.search_batch(f, a, g.nbr_ids, g.nbr_counts, cfg.alpha, QX[lo:hi], QA[lo:hi],
                                   kstar, nthreads=threads,
                                   entries=O.all_entry_points(f.shape[0], kstar, 0, hi)[lo:hi])
        return time.perf_counter() - t0, ids

    dt, _ = run(0, 4, 1)
    per = max(dt / 4, 1e-6)
    s = int(min(QX.shape[0], max(8, seconds / per)))
    dt, ids = run(0, s, 1)
    return {"value": round(s / dt, 2), "unit": UNIT, "cores": 1, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"first {s} of {QX.shape[0]} queries at K={kstar}, single thread "
                      f"(oracle/stable_oracle.c route + NumPy entry points, as search() does)",
            "parity_with_gpu_on_sample": bool(np.array_equal(ids, ids_gpu[:s]))}


# ---------------------------------------------------------------------------------------
def run_reference(args, rank, world, local):
    """The reference's CPU path (oracle port) on all host cores: the HELP build of the same
    data (timed), then bounded samples of the same queries routed at the same K*.  Nothing
    here loads the B200 library."""
    if rank != 0:
        return
    from oracle import oracle as O
    from tools.configs import OPERATING_K

    X, A, QX, QA, card = load_workload(args)
    n, m = X.shape
    l = A.shape[1]
    threads = os.cpu_count() or 1
    s_v, s_a = O.sample_statistics(X, A, min(1000, n), seed=0)
    alpha = O.compute_alpha(s_v, s_a, n, l)
    t0 = time.perf_counter()
    g = O.build(X, A, alpha, sigma=0.44, gamma=GAMMA, gamma_new=GAMMA, nthreads=0)
    build_s = time.perf_counter() - t0
    kstar = OPERATING_K.get(args.config, 100) if args.n is None else min(n, 200)
    P = max(1, kstar // 2)

    def step(lo, hi):
        ent = np.stack([O.entry_points(n, kstar, 0, qi) for qi in range(lo, hi)])
        return O.search_batch(X, A, g.nbr_ids, g.nbr_counts, alpha, QX[lo:hi], QA[lo:hi], kstar,
                              nthreads=threads, entries=ent)

    # recall at K* on a 100-query sample against the oracle's exact ground truth
    s_rec = min(100, QX.shape[0])
    ids_s, _, _ = step(0, s_rec)
    rec = float(np.mean([O.recall_at_k(ids_s[i], O.oracle_auto_topk(X, A, QX[i], QA[i], 10, alpha), 10)
                         for i in range(s_rec)]))
    t0 = time.perf_counter()
    step(0, min(QX.shape[0], 4 * threads))
    per = (time.perf_counter() - t0) / min(QX.shape[0], 4 * threads)
    budget = 150.0 / max(1, args.steps + args.warmup)
    s = int(min(QX.shape[0], max(threads, budget / max(per, 1e-6))))
    for w in range(args.warmup):
        step(0, s)
    t0 = time.perf_counter()
    for i in range(args.steps):
        lo = (i * s) % QX.shape[0]
        hi = min(QX.shape[0], lo + s)
        step(lo, hi)
    dt = (time.perf_counter() - t0) / args.steps
    value = s / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 2), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt * 1000, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args, n, m, l, card, QX.shape[0], kstar, P, X.nbytes),
        "parallelism": f"{threads} host threads",
        "recall_at_10_sample": round(rec, 4), "recall_sample_queries": s_rec,
        "build_s": round(build_s, 2),
        "build": {"cpu_s": round(build_s, 2), "cpu_threads": threads, "cpu_model": cpu_model(),
                  "iterations": g.log["iterations"], "psi_history": g.log["psi_history"],
                  "pairs": g.log["pairs"], "edges": int(g.nbr_counts.sum())},
        "cpu_baseline": {"value": round(value, 2), "unit": UNIT, "cores": threads, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": f"{s} queries per step at K={kstar}, {threads} threads "
                                   "(oracle/stable_oracle.c route + NumPy entry points) on the "
                                   "HELP graph the CPU built"},
        "e2e": {"value": round(value, 2), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world, local)
    else:
        run_mine(args, rank, world, local)


if __name__ == "__main__":
    main()

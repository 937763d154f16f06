"""Exhaustive AUTO top-k timing at a config: tensor-core path vs the fp64 SIMT path."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_01617_b200 as sb
from paper_2604_01617_b200.device import DeviceIndex
from tools.configs import make_config

X, A, QX, QA, card = make_config(os.environ.get("CFG", "cfg2"))
cfg = sb.compute_alpha(sb.sample_statistics(X, A, 1000, seed=0), X.shape[0], A.shape[1])
d = DeviceIndex(X, A, 2)
k = int(os.environ.get("K", "10"))
res = {}
for mode in os.environ.get("MODES", "1,0").split(","):
    os.environ["SB_BF_TC"] = mode
    d.bf_topk_queries(QX[:256], QA[:256], k, cfg.alpha)
    dt = 1e30
    for _ in range(int(os.environ.get("REPS", "3"))):
        t0 = time.perf_counter()
        ids, dd = d.bf_topk_queries(QX, QA, k, cfg.alpha)
        dt = min(dt, time.perf_counter() - t0)
    res[mode] = (ids, dd)
    q, n, m = QX.shape[0], X.shape[0], X.shape[1]
    flops = 2.0 * q * n * m
    print(f"SB_BF_TC={mode} {d.bf_info()} {dt*1e3:.1f} ms  {q*n/dt/1e9:.1f} G scores/s  "
          f"{flops/dt/1e12:.1f} TFLOP/s useful", flush=True)
if len(res) == 2:
    print("identical:", np.array_equal(res["1"][0], res["0"][0]) and np.array_equal(res["1"][1], res["0"][1]))

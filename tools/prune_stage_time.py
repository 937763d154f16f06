"""Time the stages of semantic_prune on the device for a config: prune_pass, reinforce_pass
(with its overflow replay) and each reconnect_islands sweep (analysis helper)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_01617_b200 as sb
from paper_2604_01617_b200 import _lib
from tools.configs import make_config

name = sys.argv[1]
X, A, QX, QA, card = make_config(name)
cfg = sb.compute_alpha(sb.sample_statistics(X, A, min(1000, X.shape[0]), seed=0), X.shape[0], A.shape[1])
schema = sb.AttributeSchema(tuple(tuple(str(i) for i in range(c)) for c in card))
p = sb.BuildParams()
g = sb.run_descent(X, A, schema, p, cfg)
dev = g.device()
t0 = time.perf_counter(); dev.prune(p.sigma); t1 = time.perf_counter()
over = ctypes.c_int64(0)
_lib.call("sb_reinforce_pass", dev.handle, float(p.sigma), ctypes.addressof(over)); dev.synchronize()
t2 = time.perf_counter()
sweeps = []
for _ in range(10):
    ran = ctypes.c_int32(0)
    ts = time.perf_counter()
    _lib.call("sb_reconnect_islands", dev.handle, float(p.sigma), ctypes.addressof(ran))
    if not ran.value:
        break
    sweeps.append(round(time.perf_counter() - ts, 3))
print(f"{name}: prune {t1 - t0:.3f}s reinforce_pass {t2 - t1:.3f}s (overflow rows {over.value}) "
      f"reconnect sweeps {sweeps}", flush=True)

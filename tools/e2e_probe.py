import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2604_01617_b200 as sb
from paper_2604_01617_b200 import _lib
from paper_2604_01617_b200.device import DeviceIndex
from tools.configs import make_config
X, A, QX, QA, card = make_config("cfg2")
cache = "/tmp/sb_graph_cfg2.npz"
if os.path.exists(cache):
    z = np.load(cache); ids, dists, counts, alpha = z["ids"], z["dists"], z["counts"], float(z["alpha"])
else:
    cfg = sb.compute_alpha(sb.sample_statistics(X, A, 1000, seed=0), X.shape[0], A.shape[1])
    g = sb.build(X, A, sb.AttributeSchema(tuple(tuple(str(i) for i in range(c)) for c in card)), sb.BuildParams(), cfg)
    ids, dists, counts, alpha = g.nbr_ids, g.nbr_dists, g.nbr_counts, cfg.alpha
    np.savez(cache, ids=ids, dists=dists, counts=counts, alpha=alpha)
dev = DeviceIndex(X, A, ids.shape[1]); dev.upload(ids, dists, counts); dev.route_prepare()
q = QX.shape[0]
qf = torch.empty((q, 128), dtype=torch.float64, pin_memory=True).numpy(); qf[:] = QX
qa = torch.empty((q, 3), dtype=torch.float64, pin_memory=True).numpy(); qa[:] = QA
os.environ["SB_ROUTE_DIRECT"] = "1"
ts = []
for i in range(8):
    t0 = time.perf_counter(); r = dev.route(qf, qa, 200, 100, 1.0 / alpha); ts.append(time.perf_counter() - t0)
print("direct-first", [round(t*1e3, 2) for t in ts], flush=True)
del os.environ["SB_ROUTE_DIRECT"]
for rep in range(2):
    ts = []
    for i in range(8):
        t0 = time.perf_counter(); r = dev.route(qf, qa, 200, 100, 1.0 / alpha); ts.append(time.perf_counter() - t0)
    print("pinned pool", [round(t*1e3, 2) for t in ts], {k: len(v) for k, v in _lib._POOL.items()}, flush=True)
# pageable outputs for comparison
orig = _lib.pinned_empty
_lib.pinned_empty = lambda shape, dtype: np.empty(shape, dtype)
ts = []
for i in range(8):
    t0 = time.perf_counter(); r = dev.route(qf, qa, 200, 100, 1.0 / alpha); ts.append(time.perf_counter() - t0)
print("pageable", [round(t*1e3, 2) for t in ts], flush=True)
_lib.pinned_empty = orig
os.environ["SB_ROUTE_DIRECT"] = "1"
ts = []
for i in range(8):
    t0 = time.perf_counter(); r = dev.route(qf, qa, 200, 100, 1.0 / alpha); ts.append(time.perf_counter() - t0)
print("direct", [round(t*1e3, 2) for t in ts], flush=True)

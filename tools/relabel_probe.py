"""Probe: how much does a locality-preserving node order speed routing up?  Builds (or loads)
the cfg index, relabels nodes by a Z-order over random projections, and times routing on the
relabeled copy against the original (same walk up to id tie-breaks)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2604_01617_b200 as sb
from paper_2604_01617_b200.device import DeviceIndex, entry_points_host
from tools.configs import make_config

cfgname = os.environ.get("CFG", "cfg2")
K = int(os.environ.get("K", "200"))
X, A, QX, QA, card = make_config(cfgname)
cache = f"/tmp/sb_graph_{cfgname}.npz"
if os.path.exists(cache):
    z = np.load(cache); ids, dists, counts, alpha = z["ids"], z["dists"], z["counts"], float(z["alpha"])
else:
    cfg = sb.compute_alpha(sb.sample_statistics(X, A, 1000, seed=0), X.shape[0], A.shape[1])
    g = sb.build(X, A, sb.AttributeSchema(tuple(tuple(str(i) for i in range(c)) for c in card)), sb.BuildParams(), cfg)
    ids, dists, counts, alpha = g.nbr_ids, g.nbr_dists, g.nbr_counts, cfg.alpha
    np.savez(cache, ids=ids, dists=dists, counts=counts, alpha=alpha)
n, m = X.shape
q = QX.shape[0]

def order_zproj(P=6, bits=10, seed=0):
    rng = np.random.default_rng(seed)
    R = rng.standard_normal((m, P)).astype(np.float32)
    Xt = torch.from_numpy(X).cuda()
    proj = (Xt @ torch.from_numpy(R).cuda()).cpu().numpy()
    lo, hi = proj.min(0), proj.max(0)
    qv = ((proj - lo) / (hi - lo + 1e-9) * ((1 << bits) - 1)).astype(np.uint64)
    key = np.zeros(n, np.uint64)
    for b in range(bits - 1, -1, -1):
        for p in range(P):
            key = (key << np.uint64(1)) | ((qv[:, p] >> np.uint64(b)) & np.uint64(1))
    return np.argsort(key, kind="stable")

def order_bfs():
    import collections
    perm = np.full(n, -1, np.int64); seen = np.zeros(n, bool); out = []
    for s in range(n):
        if seen[s]: continue
        dq = collections.deque([s]); seen[s] = True
        while dq:
            v = dq.popleft(); out.append(v)
            for u in ids[v, :counts[v]]:
                if not seen[u]: seen[u] = True; dq.append(u)
    return np.array(out)

def run(perm, label):
    inv = np.empty(n, np.int64); inv[perm] = np.arange(n)
    Xr, Ar = X[perm], A[perm]
    ids_r = np.where(np.arange(ids.shape[1])[None, :] < counts[perm][:, None], inv[ids[perm]], 0).astype(np.int32)
    dev = DeviceIndex(Xr, Ar, ids.shape[1]); dev.upload(ids_r, dists[perm], counts[perm])
    s = torch.cuda.Stream(); torch.cuda.set_stream(s); dev.set_stream(s.cuda_stream)
    qf = torch.from_numpy(QX.astype(np.float64)).cuda(); qa = torch.from_numpy(QA.astype(np.float64)).cuda()
    ent = torch.from_numpy(inv[entry_points_host(n, K, 0, 0, q)]).cuda()
    oi = torch.empty((q, K), dtype=torch.int64, device="cuda"); od = torch.empty((q, K), dtype=torch.float64, device="cuda")
    st = torch.empty((q, 5), dtype=torch.int64, device="cuda")
    f = lambda: dev.route_dev(qf.data_ptr(), qa.data_ptr(), None, q, K, K // 2, 1.0 / alpha, oi.data_ptr(), od.data_ptr(), st.data_ptr(), entries_ptr=ent.data_ptr())
    for _ in range(3): f()
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(5): f()
    e1.record(s); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    res = perm[oi.cpu().numpy()]
    print(f"{label}: {ms:.3f} ms  {q/ms*1e3:,.0f} QPS  evals={st.cpu().numpy()[:,0].mean():.0f}  orig_ids_sum={int(res.sum())}", flush=True)

run(np.arange(n), "identity")
t0 = time.time(); pz = order_zproj(); print(f"zproj order {time.time()-t0:.2f}s")
run(pz, "zproj6x10")
t0 = time.time(); pb = order_bfs(); print(f"bfs order {time.time()-t0:.2f}s")
run(pb, "bfs")

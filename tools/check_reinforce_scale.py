"""Scale check of the exact overflow path: GPU prune + reinforce + reconnect vs the CPU
oracle's prune_pass / reinforce_pass / reconnect_islands on the same post-descent graph."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_01617_b200 as sb
from paper_2604_01617_b200.device import DeviceIndex
from oracle import oracle as O
from tools.configs import make_config

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n_override = int(sys.argv[2]) if len(sys.argv) > 2 else None
X, A, QX, QA, card = make_config(name, n_override)
cfg = sb.compute_alpha(sb.sample_statistics(X, A, min(1000, X.shape[0]), seed=0), X.shape[0], A.shape[1])
schema = sb.AttributeSchema(tuple(tuple(str(i) for i in range(c)) for c in card))
p = sb.BuildParams()
t0 = time.time()
g = sb.run_descent(X, A, schema, p, cfg)
print(f"descent {time.time()-t0:.1f}s psi={g.build_log['psi_history']}", flush=True)
base = (g.nbr_ids.copy(), g.nbr_dists.copy(), g.nbr_counts.copy())
dev = DeviceIndex(X, A, p.gamma)
dev.upload(*base)
t0 = time.time(); rounds = dev.prune(p.sigma); tp = time.time() - t0
t0 = time.time(); over, sweeps = dev.reinforce(p.sigma); tr = time.time() - t0
gi, gd, gc, _ = dev.download(with_flags=False)
print(f"GPU prune {tp:.2f}s (rounds {rounds}) reinforce {tr:.2f}s overflow_rows={over} sweeps={sweeps}", flush=True)
ids, dists, counts = [x.copy() for x in base]
t0 = time.time()
indeg = O.kernels.count_in_degrees(ids, counts)
O.kernels.prune_pass(X, A, ids, dists, counts, indeg, p.sigma)
t1 = time.time()
full = O.kernels.reinforce_pass(X, A, ids, dists, counts, indeg, p.sigma)
t2 = time.time()
sw = 0
for _ in range(10):
    indeg = O.kernels.count_in_degrees(ids, counts)
    if indeg.min() >= 1: break
    O.kernels.reconnect_islands(X, A, ids, dists, counts, indeg, p.sigma); sw += 1
print(f"CPU oracle prune {t1-t0:.1f}s reinforce {t2-t1:.1f}s full_merges={full} sweeps={sw}", flush=True)
ok = np.array_equal(gc, counts) and np.array_equal(gi, ids) and np.array_equal(gd, dists)
print(f"PARITY {'OK' if ok else 'MISMATCH'}: rows differing={int((gc != counts).sum())} "
      f"ids differing={int((gi != ids).any(1).sum())} edges={int(gc.sum())}", flush=True)

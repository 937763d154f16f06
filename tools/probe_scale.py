"""Quick timing probe of the device path (not the bench): build + GT + search at a config."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_01617_b200 as sb
from tools.configs import make_config

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
n_override = int(sys.argv[2]) if len(sys.argv) > 2 else None
t0 = time.time()
X, A, QX, QA, card = make_config(name, n_override)
print(f"[{name}] data n={X.shape[0]} d={X.shape[1]} l={A.shape[1]} q={QX.shape[0]} gen {time.time()-t0:.1f}s", flush=True)
t0 = time.time()
cfg = sb.compute_alpha(sb.sample_statistics(X, A, min(1000, X.shape[0]), seed=0), X.shape[0], A.shape[1])
print(f"alpha={cfg.alpha:.6f} ({time.time()-t0:.2f}s)", flush=True)
schema = sb.AttributeSchema(tuple(tuple(str(i) for i in range(c)) for c in card))
t0 = time.time()
g = sb.build(X, A, schema, sb.BuildParams(), cfg)
bt = time.time() - t0
log = g.build_log
print(f"build {bt:.2f}s psi={log['psi_history']} init={log['seconds_init']:.2f}s iters={[round(x,2) for x in log['seconds_iterations']]} prune={log['seconds_prune']:.2f}s over={log['reinforce_overflow_rows']} rounds={log['prune_guard_rounds']} edges={int(g.nbr_counts.sum())} pairs={log.get('pairs')}", flush=True)
t0 = time.time()
gt = sb.oracle_auto_topk_batch(X, A, QX, QA, 10, cfg)
print(f"GT {time.time()-t0:.2f}s", flush=True)
for k in (10, 25, 50, 100, 200, 500, 1000):
    if k > X.shape[0]: break
    p = sb.SearchParams(k=k)
    sb.search_batch_arrays(g, QX, QA, p)
    t0 = time.time()
    ids, d, st = sb.search_batch_arrays(g, QX, QA, p)
    dt = time.time() - t0
    print(f"K={k} recall={sb.mean_recall(ids, gt):.4f} QPS(e2e wall)={QX.shape[0]/dt:,.0f} evals={st[:,0].mean():.1f}", flush=True)

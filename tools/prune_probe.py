"""Time the semantic-prune stages (prune_pass, reinforce, reconnect) on the GPU for a config."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_01617_b200 as sb
from paper_2604_01617_b200.device import DeviceIndex
from tools.configs import make_config

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
n_override = int(sys.argv[2]) if len(sys.argv) > 2 else None
X, A, QX, QA, card = make_config(name, n_override)
cfg = sb.compute_alpha(sb.sample_statistics(X, A, min(1000, X.shape[0]), seed=0), X.shape[0], A.shape[1])
schema = sb.AttributeSchema(tuple(tuple(str(i) for i in range(c)) for c in card))
p = sb.BuildParams()
t0 = time.time()
g = sb.run_descent(X, A, schema, p, cfg)
print(f"descent {time.time()-t0:.1f}s", flush=True)
dev = g.device()
t0 = time.time(); rounds = dev.prune(p.sigma); print(f"prune {time.time()-t0:.2f}s rounds {rounds}", flush=True)
t0 = time.time(); over, sweeps = dev.reinforce(p.sigma); print(f"reinforce {time.time()-t0:.2f}s overflow {over} sweeps {sweeps}", flush=True)

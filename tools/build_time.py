import os, sys, time, json
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2604_01617_b200 as sb
from tools.configs import make_config
name = sys.argv[1]
X, A, QX, QA, card = make_config(name)
cfg = sb.compute_alpha(sb.sample_statistics(X, A, 1000, seed=0), X.shape[0], A.shape[1])
schema = sb.AttributeSchema(tuple(tuple(str(i) for i in range(c)) for c in card))
t0 = time.perf_counter()
g = sb.build(X, A, schema, sb.BuildParams(), cfg)
print(name, "build_s", round(time.perf_counter() - t0, 3))
print(json.dumps({k: v for k, v in g.build_log.items()}, default=str))

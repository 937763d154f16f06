import os, sys, time, cProfile, pstats
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2604_01617_b200 as sb
from tools.configs import make_config
from cuda.bindings import runtime as rt
for sz in (1 << 28, 1 << 30, 1600 << 20):
    t0 = time.perf_counter(); e, p = rt.cudaMalloc(sz); t1 = time.perf_counter(); rt.cudaFree(p); t2 = time.perf_counter()
    print(f"cudaMalloc {sz>>20} MB {1e3*(t1-t0):.2f} ms free {1e3*(t2-t1):.2f} ms", flush=True)
X, A, QX, QA, card = make_config("cfg2")
cfg = sb.compute_alpha(sb.sample_statistics(X, A, 1000, seed=0), X.shape[0], A.shape[1])
schema = sb.AttributeSchema(tuple(tuple(str(i) for i in range(c)) for c in card))
g = sb.build(X, A, schema, sb.BuildParams(), cfg)
del g
pr = cProfile.Profile(); t0 = time.perf_counter(); pr.enable()
g = sb.build(X, A, schema, sb.BuildParams(), cfg)
pr.disable(); print("second build", time.perf_counter() - t0, {k: v for k, v in g.build_log.items() if k.startswith("seconds")})
pstats.Stats(pr).sort_stats("tottime").print_stats(22)

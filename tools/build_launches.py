"""One HELP build of a config recipe (tools/configs.py), for a per-kernel launch list under
ncu --metrics gpu__time_duration.sum: python tools/build_launches.py cfg4"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_01617_b200 as sb  # noqa: E402
from tools.configs import make_config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
X, A, QX, QA, card = make_config(name)
cfg = sb.compute_alpha(sb.sample_statistics(X, A, min(1000, X.shape[0]), seed=0), X.shape[0], A.shape[1])
schema = sb.AttributeSchema(tuple(tuple(str(i) for i in range(c)) for c in card))
t0 = time.perf_counter()
g = sb.build(X, A, schema, sb.BuildParams(), cfg)
print(name, "build", round(time.perf_counter() - t0, 3),
      {k: v for k, v in g.build_log.items() if k.startswith("seconds") or k.startswith("reinforce")}, flush=True)

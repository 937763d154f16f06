import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2604_01617_b200 as sb
from paper_2604_01617_b200.device import DeviceIndex
from tools.configs import make_config
X, A, QX, QA, card = make_config("cfg2")
cfg = sb.compute_alpha(sb.sample_statistics(X, A, 1000, seed=0), X.shape[0], A.shape[1])
schema = sb.AttributeSchema(tuple(tuple(str(i) for i in range(c)) for c in card))
p = sb.BuildParams()
g = sb.run_descent(X, A, schema, p, cfg)
dev = DeviceIndex(X, A, p.gamma)
dev.upload(g.nbr_ids, g.nbr_dists, g.nbr_counts)
dev.prune(p.sigma)
t0 = time.time(); print(dev.reinforce(p.sigma), time.time() - t0)

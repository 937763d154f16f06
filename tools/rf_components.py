"""How parallel can reinforce_pass's overflow replay be?  (analysis, not product code)

Runs descent + prune on the device for a config, downloads the pruned graph and computes, on
the host: the overflow rows O (|row_j ∪ rev_j| > gamma), their U sets, each node's exposure
(number of O rows whose U holds it) and the components of the O-row interaction graph where
rows are joined when one is in the other's U, or when they share a node p whose in-degree could
reach the safeguard (in_deg0[p] - exposure[p] < 2).  Prints sizes and per-component work.

  python tools/rf_components.py cfg5c1 [--n N]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--n", type=int, default=None)
    a = ap.parse_args()
    import scipy.sparse as sp
    from scipy.sparse.csgraph import connected_components

    import paper_2604_01617_b200 as sb
    from tools.configs import make_config
    X, A, QX, QA, card = make_config(a.config, a.n)
    n = X.shape[0]
    cfg = sb.compute_alpha(sb.sample_statistics(X, A, min(1000, n), seed=0), n, A.shape[1])
    schema = sb.AttributeSchema(tuple(tuple(str(i) for i in range(c)) for c in card))
    params = sb.BuildParams()
    g = sb.run_descent(X, A, schema, params, cfg)
    dev = g.device()
    dev.prune(params.sigma)
    ids, dists, counts, _ = dev.download(with_flags=False)
    t0 = time.perf_counter()
    G = ids.shape[1]
    src = np.repeat(np.arange(n), counts)
    mask = np.arange(G)[None, :] < counts[:, None]
    dst = ids[mask].astype(np.int64)
    # mutual edges: s -> j with s in row j
    E = sp.csr_matrix((np.ones(len(src), np.int8), (src, dst)), shape=(n, n))
    ET = E.T.tocsr()
    mutual = E.multiply(ET)
    rev_extra = np.asarray((ET - mutual).sum(axis=1)).ravel()  # reverse sources row j lacks
    indeg0 = np.asarray(ET.sum(axis=1)).ravel()
    O = np.nonzero(counts + rev_extra > G)[0]
    print(f"{a.config}: n={n} edges={len(src)} O rows={len(O)}")
    if len(O) == 0:
        return
    # U_j = row_j ∪ rev_j for j in O, as a sparse O x n membership matrix
    U = (E + ET)[O].tocsr()
    U.data[:] = 1
    exposure = np.asarray(U.sum(axis=0)).ravel()
    unsafe = (indeg0 - exposure) < 2
    print(f"  U sizes: mean {U.getnnz(axis=1).mean():.1f} max {U.getnnz(axis=1).max()}; "
          f"unsafe nodes {int(unsafe.sum())} (exposed {int((exposure > 0).sum())})")
    no = len(O)
    oidx = -np.ones(n, np.int64)
    oidx[O] = np.arange(no)
    # (a) O rows inside other O rows' U
    Ucoo = U.tocoo()
    inO = oidx[Ucoo.col] >= 0
    r1, c1 = Ucoo.row[inO], oidx[Ucoo.col[inO]]
    # (b) O rows sharing an unsafe node: link every row holding p to the first row holding p
    Uu = U[:, np.nonzero(unsafe)[0]].tocsc()
    r2, c2 = [], []
    for k in range(Uu.shape[1]):
        rows = Uu.indices[Uu.indptr[k]:Uu.indptr[k + 1]]
        if len(rows) > 1:
            r2.append(rows[1:])
            c2.append(np.full(len(rows) - 1, rows[0]))
    r2 = np.concatenate(r2) if r2 else np.zeros(0, np.int64)
    c2 = np.concatenate(c2) if c2 else np.zeros(0, np.int64)
    rr = np.concatenate([r1, r2])
    cc = np.concatenate([c1, c2])
    Gi = sp.csr_matrix((np.ones(len(rr), np.int8), (rr, cc)), shape=(no, no))
    ncomp, lab = connected_components(Gi, directed=False)
    sizes = np.bincount(lab)
    work = np.bincount(lab, weights=U.getnnz(axis=1))
    order = np.argsort(-work)
    print(f"  interaction edges: in-U {len(r1)}, unsafe-shared {len(r2)}")
    print(f"  components {ncomp}; largest by rows {sizes.max()} ({sizes.max() / no:.1%}); "
          f"largest by U work {work.max():.0f} of {work.sum():.0f} ({work.max() / work.sum():.1%})")
    print("  top components (rows, U work):", [(int(sizes[i]), int(work[i])) for i in order[:8]])
    # the same without the unsafe-sharing links (in-U only)
    G1 = sp.csr_matrix((np.ones(len(r1), np.int8), (r1, c1)), shape=(no, no))
    n1, l1 = connected_components(G1, directed=False)
    w1 = np.bincount(l1, weights=U.getnnz(axis=1))
    print(f"  in-U links only: components {n1}, largest work share {w1.max() / w1.sum():.1%}")
    print(f"  analysis {time.perf_counter() - t0:.1f} s")


if __name__ == "__main__":
    main()

"""Multi-process (world_size 2, gloo, CPU) tests of the sharded hot path:
query-sharded routing and node-sharded exact top-k with one exchange step.  The per-shard
compute is the CPU oracle here (no GPU in CI); the sharding, global query indices, gather
order and (dist, id) merge are the code under test."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2604_01617_b200 import sharding


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _data(seed=5, n=700, m=12, l=2, q=23):
    rng = np.random.default_rng(seed)
    f = rng.standard_normal((n, m)).astype(np.float32)
    a = rng.integers(1, 4, (n, l)).astype(np.int32)
    qf = rng.standard_normal((q, m)).astype(np.float32)
    qa = rng.integers(1, 4, (q, l)).astype(np.int32)
    return f, a, qf, qa


def _oracle_route(f, a, ids, cnt, alpha, k, seed):
    n = f.shape[0]

    def route_fn(qf, qa, masks, qi0):
        ent = np.stack([O.entry_points(n, k, seed, qi0 + i) for i in range(qf.shape[0])])
        return O.route_batch_raw(f, a, ids, cnt, qf, qa, masks, 1.0 / alpha, ent, max(1, k // 2),
                                 True, 1)
    return route_fn


def _oracle_local_topk(alpha):
    def local_fn(f, a, qf, qa, kk, masks):
        out_i = np.empty((qf.shape[0], kk), np.int64)
        out_d = np.empty((qf.shape[0], kk), np.float64)
        for i in range(qf.shape[0]):
            m = None if masks is None else masks[i]
            out_i[i], out_d[i] = O.oracle_auto_topk(f, a, qf[i], qa[i], kk, alpha, m, return_dists=True)
        return out_i, out_d
    return local_fn


class _OracleDevice:
    """CPU stand-in for DeviceIndex.route_dev: same pointer-based contract (row block of the
    query tensors in, results written through the output pointers), oracle compute."""

    def __init__(self, f, a, ids, cnt, alpha, k, seed):
        self.f, self.a, self.ids, self.cnt, self.alpha, self.k, self.seed = f, a, ids, cnt, alpha, k, seed

    def set_stream(self, s):
        raise AssertionError("CPU tensors need no stream")

    def route_dev(self, qf_ptr, qa_ptr, qm_ptr, q, k, pioneer, inv_alpha, ids_ptr, dists_ptr,
                  stats_ptr=None, entries_ptr=None, seed=0, qi0=0, use_coarse=True):
        import ctypes
        m, l = self.f.shape[1], self.a.shape[1]
        view = lambda p, t, shape: np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(t)), shape)
        qf = view(qf_ptr, ctypes.c_double, (q, m)).copy()
        qa = view(qa_ptr, ctypes.c_double, (q, l)).copy()
        ent = np.stack([O.entry_points(self.f.shape[0], k, seed, qi0 + i) for i in range(q)])
        i, d, st = O.route_batch_raw(self.f, self.a, self.ids, self.cnt, qf, qa, None,
                                     inv_alpha, ent, pioneer, use_coarse, 1)
        view(ids_ptr, ctypes.c_int64, (q, k))[:] = i
        view(dists_ptr, ctypes.c_double, (q, k))[:] = d
        view(stats_ptr, ctypes.c_int64, (q, 5))[:, :4] = st


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        f, a, qf, qa = _data()
        alpha = 1.07
        g = O.build(f, a, alpha, gamma=24, gamma_new=24)
        k, seed = 16, 3
        got = sharding.search_batch_sharded(None, qf, qa, None,
                                            route_fn=_oracle_route(f, a, g.nbr_ids, g.nbr_counts,
                                                                   alpha, k, seed))
        ti, td = sharding.oracle_auto_topk_sharded(f, a, qf, qa, 9, None,
                                                   local_fn=_oracle_local_topk(alpha))
        import torch
        dev = _OracleDevice(f, a, g.nbr_ids, g.nbr_counts, alpha, k, seed)
        qf_t = torch.from_numpy(np.ascontiguousarray(qf, np.float64))
        qa_t = torch.from_numpy(np.ascontiguousarray(qa, np.float64))
        di, dd, ds = sharding.search_batch_sharded_device(dev, qf_t, qa_t, qf.shape[0], k,
                                                          max(1, k // 2), 1.0 / alpha, seed=seed)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), ids=got[0], dists=got[1], stats=got[2],
                 ti=ti, td=td, dev_ids=di.numpy(), dev_dists=dd.numpy(),
                 dev_stats=ds.numpy()[:, :4])
    finally:
        dist.destroy_process_group()


def test_shard_range_partitions():
    for total in (0, 1, 7, 100, 101):
        for world in (1, 2, 3, 8):
            spans = [sharding.shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def test_merge_topk_orders_by_dist_then_id():
    d = [np.array([[1.0, 2.0, np.inf]]), np.array([[1.0, 0.5, 3.0]])]
    i = [np.array([[7, 3, 2**62]]), np.array([[4, 9, 1]])]
    ids, dists = sharding.merge_topk(d, i, 4)
    np.testing.assert_array_equal(ids, [[9, 4, 7, 3]])
    np.testing.assert_array_equal(dists, [[0.5, 1.0, 1.0, 2.0]])


def test_single_process_is_identity():
    f, a, qf, qa = _data(n=300, q=7)
    alpha = 1.07
    ti, td = sharding.oracle_auto_topk_sharded(f, a, qf, qa, 5, None,
                                               local_fn=_oracle_local_topk(alpha))
    for i in range(qf.shape[0]):
        wi, wd = O.oracle_auto_topk(f, a, qf[i], qa[i], 5, alpha, return_dists=True)
        np.testing.assert_array_equal(ti[i], wi)
        np.testing.assert_array_equal(td[i], wd)


@pytest.mark.timeout(300)
def test_two_ranks_gloo_match_single_process(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    f, a, qf, qa = _data()
    alpha = 1.07
    g = O.build(f, a, alpha, gamma=24, gamma_new=24)
    want = O.search_batch(f, a, g.nbr_ids, g.nbr_counts, alpha, qf, qa, 16, seed=3)
    wi = np.empty((qf.shape[0], 9), np.int64)
    wd = np.empty((qf.shape[0], 9), np.float64)
    for i in range(qf.shape[0]):
        wi[i], wd[i] = O.oracle_auto_topk(f, a, qf[i], qa[i], 9, alpha, return_dists=True)
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        np.testing.assert_array_equal(z["ids"], want[0])
        np.testing.assert_array_equal(z["dists"], want[1])
        np.testing.assert_array_equal(z["stats"], want[2])
        np.testing.assert_array_equal(z["ti"], wi)
        np.testing.assert_array_equal(z["td"], wd)
        np.testing.assert_array_equal(z["dev_ids"], want[0])
        np.testing.assert_array_equal(z["dev_dists"], want[1])
        np.testing.assert_array_equal(z["dev_stats"], want[2])


@pytest.mark.gpu
def test_sharded_defaults_run_the_b200_path():
    """Single process, default compute = the CUDA library: equal to the unsharded calls."""
    import paper_2604_01617_b200 as sb
    f, a, qf, qa = _data(n=2000, q=40)
    cfg = sb.MetricConfig.manual(1.07, a.shape[1])
    ti, td = sharding.oracle_auto_topk_sharded(f, a, qf, qa, 10, cfg)
    wi, wd = sb.oracle_auto_topk_batch(f, a, qf, qa, 10, cfg, return_dists=True)
    np.testing.assert_array_equal(ti, wi)
    np.testing.assert_array_equal(td, wd)
    schema = sb.AttributeSchema(tuple(tuple(str(i) for i in range(4)) for _ in range(a.shape[1])))
    g = sb.build(f, a, schema, sb.BuildParams(gamma=24, gamma_new=24), cfg)
    p = sb.SearchParams(k=16, seed=3)
    got = sharding.search_batch_sharded(g, qf, qa, p)
    want = sb.search_batch_arrays(g, qf, qa, p)
    for x, y in zip(got, want):
        np.testing.assert_array_equal(x, y)


@pytest.mark.gpu
def test_device_sharded_routing_single_process():
    """search_batch_sharded_device on one GPU equals the public search_batch."""
    import torch
    import paper_2604_01617_b200 as sb
    f, a, qf, qa = _data(n=3000, q=50)
    cfg = sb.MetricConfig.manual(1.07, a.shape[1])
    schema = sb.AttributeSchema(tuple(tuple(str(i) for i in range(4)) for _ in range(a.shape[1])))
    g = sb.build(f, a, schema, sb.BuildParams(gamma=24, gamma_new=24), cfg)
    p = sb.SearchParams(k=20, seed=2)
    want = sb.search_batch_arrays(g, qf, qa, p)
    qf_d = torch.from_numpy(np.ascontiguousarray(qf, np.float64)).cuda()
    qa_d = torch.from_numpy(np.ascontiguousarray(qa, np.float64)).cuda()
    got = sharding.search_batch_sharded_device(g.device(), qf_d, qa_d, qf.shape[0], 20, 10,
                                               1.0 / 1.07, seed=2)
    torch.cuda.synchronize()
    g.device().set_stream(None)
    for x, y in zip(got, want):
        np.testing.assert_array_equal(x.cpu().numpy(), y)

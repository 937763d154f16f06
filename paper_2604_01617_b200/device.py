"""DeviceIndex: one C-ABI index handle (dataset + adjacency resident in HBM)."""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import c64, ptr


class DeviceIndex:
    """Owns an ``sb_index``: features f32[n,m], attrs i32[n,l], adjacency of capacity gamma."""

    def __init__(self, features: np.ndarray, attrs: np.ndarray, gamma: int):
        _lib.require_gpu()
        self.features = c64(features, np.float32)
        self.attrs = c64(attrs, np.int32)
        if self.features.ndim != 2 or self.attrs.ndim != 2:
            raise ValueError("features and attrs must be 2-D")
        if self.features.shape[0] != self.attrs.shape[0]:
            raise ValueError("features and attrs disagree on n")
        self.n, self.m = self.features.shape
        self.l = self.attrs.shape[1]
        self.gamma = int(gamma)
        h = ctypes.c_void_p(0)
        _lib.call("sb_index_create", ptr(self.features), ptr(self.attrs), self.n, self.m, self.l,
                  self.gamma, ctypes.byref(h))
        self._h = h

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.load().sb_index_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- adjacency -----------------------------------------------------------------
    def upload(self, ids, dists, counts, flags=None):
        ids = c64(ids, np.int32)
        dists = c64(dists, np.float32)
        counts = c64(counts, np.int32)
        fl = None if flags is None else c64(flags, np.uint8)
        if ids.shape != (self.n, self.gamma) or dists.shape != ids.shape:
            raise ValueError("adjacency shape mismatch")
        _lib.call("sb_adj_upload", self._h, ptr(ids), ptr(dists), ptr(counts), ptr(fl))

    def download(self, with_flags=True):
        ids = np.empty((self.n, self.gamma), np.int32)
        dists = np.empty((self.n, self.gamma), np.float32)
        counts = np.empty(self.n, np.int32)
        flags = np.empty((self.n, self.gamma), np.uint8) if with_flags else None
        _lib.call("sb_adj_download", self._h, ptr(ids), ptr(dists), ptr(counts), ptr(flags))
        return ids, dists, counts, flags

    def set_stream(self, stream_ptr: int | None):
        _lib.call("sb_set_stream", self._h, stream_ptr)

    def synchronize(self):
        _lib.call("sb_synchronize", self._h)

    def launch_count(self) -> int:
        return int(_lib.load().sb_launch_count(self._h))

    def info(self) -> dict:
        ie = ctypes.c_int32(0)
        fm = ctypes.c_double(0.0)
        tc = ctypes.c_int32(0)
        _lib.call("sb_index_info", self._h, ctypes.addressof(ie), ctypes.addressof(fm),
                  ctypes.addressof(tc))
        return {"int_exact": bool(ie.value), "fmax_abs": fm.value, "last_bf_tc": bool(tc.value)}

    def route_info(self) -> dict:
        """Distance path of the last routing launch and the feature bytes it reads per row."""
        path = ctypes.c_int32(-1)
        rb = ctypes.c_int32(0)
        _lib.call("sb_route_info", self._h, ctypes.addressof(path), ctypes.addressof(rb))
        names = {0: "fp64", 1: "fp32", 2: "fp32-groups", 3: "fp64-generic", 4: "u8-dp4a",
                 5: "fp32-filter+fp64", 6: "fp64"}
        return {"path": names.get(path.value, "none"), "row_bytes": rb.value,
                "pipelined": path.value == 6}

    def bf_info(self) -> dict:
        """Path of the last exhaustive top-k call, TF32 candidates passed to the re-rank and
        queries recomputed on the fp64 kernel (sb_bf_info)."""
        path = ctypes.c_int32(-1)
        cands = ctypes.c_int64(0)
        fb = ctypes.c_int64(0)
        ms = ctypes.c_double(0.0)
        _lib.call("sb_bf_info", self._h, ctypes.addressof(path), ctypes.addressof(cands),
                  ctypes.addressof(fb), ctypes.addressof(ms))
        names = {0: "fp64", 1: "tc-int-exact", 2: "tc-tf32-filter"}
        return {"path": names.get(path.value, "none"), "candidates": cands.value,
                "fallback_queries": fb.value, "kernel_ms": ms.value}

    def route_prepare(self):
        """Build the routing layout (locality order, u8 copy) now; see sb_route_prepare."""
        _lib.call("sb_route_prepare", self._h)

    def set_distance_mode(self, sequential: bool):
        _lib.call("sb_set_distance_mode", self._h, 1 if sequential else 0)

    # ---- HELP build ------------------------------------------------------------------
    def init_graph(self, ids, inv_alpha: float):
        """Initial distances/flags/counts; ids = None keeps the rows already on the device."""
        ids = None if ids is None else c64(ids, np.int32)
        _lib.call("sb_init_graph", self._h, ptr(ids), float(inv_alpha))

    def init_random_ids(self, seed: int):
        """graph.py:120-123 on the device; returns (32-bit draws consumed, the buffered high
        half NumPy keeps when that count is odd, rows to redraw)."""
        consumed = ctypes.c_int64(0)
        buf = ctypes.c_uint32(0)
        nbad = ctypes.c_int64(0)
        _lib.call("sb_init_random_ids", self._h, int(seed), ctypes.addressof(consumed),
                  ctypes.addressof(buf), None, 0, ctypes.addressof(nbad))
        bad = np.empty(max(1, nbad.value), np.int64)
        if nbad.value:
            _lib.call("sb_init_random_ids", self._h, int(seed), ctypes.addressof(consumed),
                      ctypes.addressof(buf), ptr(bad), bad.shape[0], ctypes.addressof(nbad))
        return consumed.value, buf.value, bad[: nbad.value]

    def set_rows(self, rows: np.ndarray, ids: np.ndarray):
        rows = c64(rows, np.int64)
        ids = c64(ids, np.int32)
        if ids.shape != (rows.shape[0], self.gamma):
            raise ValueError("ids must be len(rows) x gamma")
        _lib.call("sb_set_rows", self._h, ptr(rows), rows.shape[0], ptr(ids))

    def build_candidates(self, gamma_new: int, download=False):
        if not download:
            _lib.call("sb_build_candidates", self._h, int(gamma_new), None, None, None, None)
            return None
        nc = np.empty((self.n, gamma_new), np.int32)
        ncnt = np.empty(self.n, np.int32)
        oc = np.empty((self.n, self.gamma), np.int32)
        ocnt = np.empty(self.n, np.int32)
        _lib.call("sb_build_candidates", self._h, int(gamma_new), ptr(nc), ptr(ncnt), ptr(oc),
                  ptr(ocnt))
        return nc, ncnt, oc, ocnt

    def local_join(self, inv_alpha: float):
        ins = ctypes.c_int64(0)
        pairs = ctypes.c_int64(0)
        _lib.call("sb_local_join", self._h, float(inv_alpha), ctypes.addressof(ins),
                  ctypes.addressof(pairs))
        return ins.value, pairs.value

    def descent_iteration(self, gamma_new: int, inv_alpha: float):
        ins = ctypes.c_int64(0)
        pairs = ctypes.c_int64(0)
        _lib.call("sb_descent_iteration", self._h, int(gamma_new), float(inv_alpha),
                  ctypes.addressof(ins), ctypes.addressof(pairs))
        return ins.value, pairs.value

    def count_in_degrees(self) -> np.ndarray:
        out = np.empty(self.n, np.int64)
        _lib.call("sb_count_in_degrees", self._h, ptr(out))
        return out

    def get_rows(self, rows: np.ndarray):
        rows = c64(rows, np.int64)
        ids = np.empty((rows.shape[0], self.gamma), np.int32)
        counts = np.empty(rows.shape[0], np.int32)
        _lib.call("sb_get_rows", self._h, ptr(rows), rows.shape[0], ptr(ids), ptr(counts))
        return ids, counts

    def prune(self, sigma: float) -> int:
        rounds = ctypes.c_int32(0)
        _lib.call("sb_prune", self._h, float(sigma), ctypes.addressof(rounds))
        return rounds.value

    def reinforce(self, sigma: float):
        over = ctypes.c_int64(0)
        sweeps = ctypes.c_int32(0)
        _lib.call("sb_reinforce", self._h, float(sigma), ctypes.addressof(over),
                  ctypes.addressof(sweeps))
        return over.value, sweeps.value

    # ---- exhaustive top-k --------------------------------------------------------------
    def bf_topk_nodes(self, sample_ids: np.ndarray, k: int, inv_alpha: float) -> np.ndarray:
        s = c64(sample_ids, np.int64)
        out = np.empty((s.shape[0], k), np.int32)
        _lib.call("sb_bf_topk_nodes", self._h, ptr(s), s.shape[0], int(k), float(inv_alpha),
                  ptr(out))
        return out

    def bf_topk_queries(self, qf, qa, k: int, alpha: float, qmask=None):
        qf = c64(np.atleast_2d(qf), np.float64)
        qa = c64(np.atleast_2d(qa), np.int64)
        qm = None if qmask is None else c64(np.atleast_2d(qmask), np.int64)
        q = qf.shape[0]
        if qf.shape[1] != self.m or qa.shape != (q, self.l):
            raise ValueError("query shape mismatch")
        ids = np.empty((q, k), np.int64)
        dists = np.empty((q, k), np.float64)
        unc = ctypes.c_int32(0)
        _lib.call("sb_bf_topk_queries", self._h, ptr(qf), ptr(qa), ptr(qm), q, int(k),
                  float(alpha), ptr(ids), ptr(dists), ctypes.addressof(unc))
        if unc.value:
            raise RuntimeError(f"{unc.value} queries could not be certified exact (tie cluster "
                               "wider than the re-rank margin)")
        return ids, dists

    def hybrid_groundtruth(self, qf, qa, k: int, qmask=None):
        """oracle_hybrid_groundtruth (evaluate.py:58-77) for q queries: (ids q x k padded with
        -1, pure feature distances q x k, per-query counts = min(k, matches))."""
        qf = c64(np.atleast_2d(qf), np.float64)
        qa = c64(np.atleast_2d(qa), np.int64)
        qm = None if qmask is None else c64(np.atleast_2d(qmask), np.int64)
        q = qf.shape[0]
        if qf.shape[1] != self.m or qa.shape != (q, self.l):
            raise ValueError("query shape mismatch")
        ids = np.empty((q, k), np.int64)
        dists = np.empty((q, k), np.float64)
        counts = np.empty(q, np.int64)
        _lib.call("sb_hybrid_groundtruth", self._h, ptr(qf), ptr(qa), ptr(qm), q, int(k),
                  ptr(ids), ptr(dists), ptr(counts))
        return ids, dists, counts

    # ---- routing -----------------------------------------------------------------------
    def route(self, qf, qa, k: int, pioneer: int, inv_alpha: float, qmask=None, entries=None,
              seed: int = 0, qi0: int = 0, use_coarse: bool = True, stats=True):
        qf = c64(np.atleast_2d(qf), np.float64)
        qa = c64(np.atleast_2d(qa), np.float64)
        qm = None if qmask is None else c64(np.atleast_2d(qmask), np.float64)
        ent = None if entries is None else c64(np.atleast_2d(entries), np.int64)
        q = qf.shape[0]
        ids = _lib.pinned_empty((q, k), np.int64)
        dists = _lib.pinned_empty((q, k), np.float64)
        st = _lib.pinned_empty((q, 5), np.int64) if stats else None
        _lib.call("sb_route_batch", self._h, ptr(qf), ptr(qa), ptr(qm), q, int(k), int(pioneer),
                  1 if use_coarse else 0, ptr(ent), int(seed), int(qi0), float(inv_alpha),
                  ptr(ids), ptr(dists), ptr(st))
        return ids, dists, st

    def route_dev(self, qf_ptr, qa_ptr, qm_ptr, q: int, k: int, pioneer: int, inv_alpha: float,
                  ids_ptr, dists_ptr, stats_ptr=None, entries_ptr=None, seed: int = 0,
                  qi0: int = 0, use_coarse: bool = True):
        """All pointers are device pointers (e.g. torch tensor data_ptr()); asynchronous."""
        _lib.call("sb_route_batch_dev", self._h, qf_ptr, qa_ptr, qm_ptr, int(q), int(k),
                  int(pioneer), 1 if use_coarse else 0, entries_ptr, int(seed), int(qi0),
                  float(inv_alpha), ids_ptr, dists_ptr, stats_ptr)


def entry_points_host(n: int, k: int, seed: int, qi0: int, q: int) -> np.ndarray:
    """router.py:42-45 for q consecutive query indices, via the C port (no GPU needed)."""
    out = np.empty((q, k), np.int64)
    _lib.call("sb_entry_points", int(n), int(k), int(seed), int(qi0), int(q), ptr(out))
    return out


def entry_points_device(n: int, k: int, seed: int, qi0: int, q: int) -> np.ndarray:
    """entry_points (router.py:42-45) for queries qi0 .. qi0 + q - 1 drawn by the device kernels
    that routing uses (warp-parallel Floyd draws, shared-memory tables), copied back."""
    out = np.empty((q, k), np.int64)
    _lib.call("sb_entry_points_device", int(n), int(k), int(seed), int(qi0), int(q), ptr(out))
    return out

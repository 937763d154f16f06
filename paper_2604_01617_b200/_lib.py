"""ctypes binding of libstable_b200.so (C ABI: include/stable_b200.h).

The shared library is built in-tree (``make -C paper_2604_01617_b200`` or
``__graft_entry__.build()``).  There is no fallback: if the library is missing or no CUDA
device is visible, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import ConstraintError, FormatError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("STABLE_B200_LIB") or os.path.join(_HERE, "libstable_b200.so")

SB_OK, SB_EARG, SB_EFORMAT, SB_ECONSTRAINT, SB_ECUDA = 0, 1, 2, 3, 4

_i32, _i64, _u64, _f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
_vp = ctypes.c_void_p
_pp = ctypes.POINTER(ctypes.c_void_p)

# name -> argtypes (all return int unless listed in _RESTYPE)
_SIGS = {
    "sb_last_error": [],
    "sb_version": [],
    "sb_device_count": [_vp],
    "sb_index_create": [_vp, _vp, _i64, _i32, _i32, _i32, _pp],
    "sb_index_destroy": [_vp],
    "sb_set_stream": [_vp, _vp],
    "sb_synchronize": [_vp],
    "sb_adj_upload": [_vp, _vp, _vp, _vp, _vp],
    "sb_adj_download": [_vp, _vp, _vp, _vp, _vp],
    "sb_init_graph": [_vp, _vp, _f64],
    "sb_init_random_ids": [_vp, _u64, _vp, _vp, _vp, _i64, _vp],
    "sb_set_rows": [_vp, _vp, _i64, _vp],
    "sb_build_candidates": [_vp, _i32, _vp, _vp, _vp, _vp],
    "sb_set_candidates": [_vp, _i32, _vp, _vp, _vp, _vp],
    "sb_local_join": [_vp, _f64, _vp, _vp],
    "sb_descent_iteration": [_vp, _i32, _f64, _vp, _vp],
    "sb_count_in_degrees": [_vp, _vp],
    "sb_get_rows": [_vp, _vp, _i64, _vp, _vp],
    "sb_prune": [_vp, _f64, _vp],
    "sb_reinforce": [_vp, _f64, _vp, _vp],
    "sb_reinforce_pass": [_vp, _f64, _vp],
    "sb_reconnect_islands": [_vp, _f64, _vp],
    "sb_bf_topk_nodes": [_vp, _vp, _i64, _i32, _f64, _vp],
    "sb_bf_topk_queries": [_vp, _vp, _vp, _vp, _i64, _i32, _f64, _vp, _vp, _vp],
    "sb_hybrid_groundtruth": [_vp, _vp, _vp, _vp, _i64, _i32, _vp, _vp, _vp],
    "sb_entry_points": [_i64, _i32, _u64, _i64, _i64, _vp],
    "sb_entry_points_device": [_i64, _i32, _u64, _i64, _i64, _vp],
    "sb_route_batch": [_vp, _vp, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _u64, _i64, _f64,
                       _vp, _vp, _vp],
    "sb_route_batch_dev": [_vp, _vp, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _u64, _i64, _f64,
                           _vp, _vp, _vp],
    "sb_launch_count": [_vp],
    "sb_index_info": [_vp, _vp, _vp, _vp],
    "sb_set_distance_mode": [_vp, _i32],
    "sb_route_info": [_vp, _vp, _vp],
    "sb_bf_info": [_vp, _vp, _vp, _vp, _vp],
    "sb_route_prepare": [_vp],
    "sb_host_alloc": [ctypes.c_size_t, _pp],
    "sb_host_free": [_vp],
}
_RESTYPE = {"sb_last_error": ctypes.c_char_p, "sb_launch_count": ctypes.c_int64}

_LIB = None


def load():
    """Load the shared library (raises if it was not built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()')")
        lib = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPE.get(name, ctypes.c_int)
        _LIB = lib
    return _LIB


def exported_symbols():
    return list(_SIGS)


def check(rc: int) -> None:
    if rc == SB_OK:
        return
    msg = load().sb_last_error().decode(errors="replace")
    if rc == SB_EARG:
        raise ValueError(msg)
    if rc == SB_EFORMAT:
        raise FormatError(msg)
    if rc == SB_ECONSTRAINT:
        raise ConstraintError(msg)
    raise RuntimeError(f"CUDA error in libstable_b200: {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def device_count() -> int:
    c = ctypes.c_int(0)
    rc = load().sb_device_count(ctypes.addressof(c))
    return c.value if rc == SB_OK else 0


def require_gpu() -> None:
    if device_count() < 1:
        raise RuntimeError("no CUDA device visible: the B200 path has no CPU fallback")


# ---- page-locked result buffers ----------------------------------------------------------
# Results come back through pinned memory (full-speed, asynchronous D2H).  Blocks are recycled:
# a returned array owns its block until it (and every view of it) is garbage collected.
_POOL: dict[int, list[int]] = {}


def _release(nbytes: int, addr: int) -> None:
    _POOL.setdefault(nbytes, []).append(addr)


def pinned_empty(shape, dtype) -> np.ndarray:
    """np.empty in page-locked host memory."""
    import weakref
    dt = np.dtype(dtype)
    count = int(np.prod(shape))
    nbytes = max(64, ((count * dt.itemsize + 4095) // 4096) * 4096)
    free = _POOL.get(nbytes)
    if free:
        addr = free.pop()
    else:
        p = ctypes.c_void_p(0)
        check(load().sb_host_alloc(nbytes, ctypes.byref(p)))
        addr = p.value
    buf = (ctypes.c_char * nbytes).from_address(addr)
    # The block goes back to the pool only when the ctypes buffer dies: every array that
    # reads it (the frombuffer base, its reshape, any row view handed to a caller) holds a
    # reference chain to `buf`, so a block is never recycled while a result still uses it.
    weakref.finalize(buf, _release, nbytes, addr)
    return np.frombuffer(buf, dtype=dt, count=count).reshape(shape)


def fingerprint(a: np.ndarray) -> tuple:
    """Content fingerprint of a host array (shape, dtype, xor and wrapping sum of its words).

    The device caches key on it, so a cache hit needs the same contents, not just the same
    buffer address: an array written in place, or a new array that lands on a freed address,
    re-uploads.  Costs one read of the array (≈0.1 s for 512 MB)."""
    a = np.ascontiguousarray(a)
    raw = a.reshape(-1).view(np.uint8)
    head = raw[: raw.size - raw.size % 8].view(np.uint64)
    tail = bytes(raw[raw.size - raw.size % 8:])
    return (a.shape, a.dtype.str, int(np.bitwise_xor.reduce(head)) if head.size else 0,
            int(np.add.reduce(head)) if head.size else 0, tail)


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data


def c64(a, dtype) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dtype)

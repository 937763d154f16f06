"""HELP relation-graph construction on the B200 (reference graph.py:22-280) and the "HELP"
v1 index format (reference graph.py:287-415).

Orchestration stays thin host Python, exactly the reference's sequence of steps; every bulk
step runs on the device through the C ABI:

  init_random_graph   host NumPy ids (graph.py:120-129; duplicate rows resampled with an
                      O(gamma) stream-identical rewrite) -> sb_init_graph (distances + sort)
  quality estimate    host NumPy sample (graph.py:182-184) -> sb_bf_topk_nodes
  psi                 sb_get_rows of the sample, summed on the host in the reference's order
  descent_iteration   sb_descent_iteration (candidates + local join)
  semantic_prune      sb_prune (Jacobi-guard prune) + sb_reinforce (symmetrise / exact replay
                      + reconnect sweeps)

During run_descent the adjacency stays on the device; the host arrays are refreshed when a
public step returns.
"""

from __future__ import annotations

import struct
import time
from dataclasses import dataclass, field

import numpy as np

from .device import DeviceIndex
from .errors import FormatError
from .metric import AttributeSchema, MetricConfig, SampleStats

INDEX_MAGIC = b"HELP"
INDEX_VERSION = 1


@dataclass
class BuildParams:
    """Knobs of graph construction (reference graph.py:22-47)."""

    gamma: int = 100
    gamma_new: int = 100
    sigma: float = 0.44
    psi_target: float = 0.8
    max_iterations: int = 30
    quality_sample: int = 100
    quality_k: int | None = None
    seed: int = 0

    def __post_init__(self):
        if self.gamma < 2:
            raise ValueError("gamma must be >= 2")
        if self.gamma_new < 1:
            raise ValueError("gamma_new must be >= 1")
        if not 0 <= self.psi_target <= 1:
            raise ValueError("psi_target must be in [0, 1]")
        if not -1 <= self.sigma <= 1:
            raise ValueError("sigma must be in [-1, 1]")
        if self.quality_sample < 1:
            raise ValueError("quality_sample must be >= 1")
        if self.quality_k is not None and self.quality_k < 1:
            raise ValueError("quality_k must be >= 1")


@dataclass
class QualityEstimate:
    sample_ids: np.ndarray
    ground_truth: np.ndarray
    psi: float = 0.0


@dataclass
class RelationGraph:
    """Fixed-capacity adjacency sorted by fused distance (reference graph.py:60-103)."""

    features: np.ndarray
    attrs: np.ndarray
    schema: AttributeSchema
    metric: MetricConfig
    sigma: float
    nbr_ids: np.ndarray
    nbr_dists: np.ndarray
    nbr_counts: np.ndarray
    nbr_flags: np.ndarray | None = None
    frozen: bool = False
    build_log: dict = field(default_factory=dict)
    quality: QualityEstimate | None = None
    # device mirror; `_dev_sync` is True when its adjacency equals the host arrays
    _device: DeviceIndex | None = field(default=None, repr=False, compare=False)
    _dev_sync: bool = field(default=False, repr=False, compare=False)

    @property
    def n(self) -> int:
        return self.features.shape[0]

    @property
    def gamma(self) -> int:
        return self.nbr_ids.shape[1]

    def device(self) -> DeviceIndex:
        """The device index holding this graph's adjacency (uploaded on first use)."""
        d = self._device
        if d is None or d.n != self.n or d.gamma != self.gamma:
            d = DeviceIndex(self.features, self.attrs, self.gamma)
            self._device = d
            self._dev_sync = False
        if not self._dev_sync:
            d.upload(self.nbr_ids, self.nbr_dists, self.nbr_counts, self.nbr_flags)
            self._dev_sync = True
        return d

    def _pull(self):
        ids, dists, counts, flags = self._device.download(with_flags=self.nbr_flags is not None)
        self.nbr_ids, self.nbr_dists, self.nbr_counts = ids, dists, counts
        if self.nbr_flags is not None:
            self.nbr_flags = flags
        self._dev_sync = True

    def in_degrees(self) -> np.ndarray:
        """count_in_degrees (_kernels.py:256-263)."""
        return self.device().count_in_degrees()

    def copy_unfrozen(self) -> "RelationGraph":
        return RelationGraph(
            features=self.features, attrs=self.attrs, schema=self.schema, metric=self.metric,
            sigma=self.sigma, nbr_ids=self.nbr_ids.copy(), nbr_dists=self.nbr_dists.copy(),
            nbr_counts=self.nbr_counts.copy(),
            nbr_flags=None if self.nbr_flags is None else self.nbr_flags.copy(),
            frozen=False, build_log=dict(self.build_log), quality=self.quality)


# ---------------------------------------------------------------------------
def init_random_ids(n: int, gamma: int, seed: int) -> np.ndarray:
    """The reference's random neighbour ids (graph.py:120-129), same NumPy stream.

    Duplicate rows are redrawn with rng.choice(n - 1, gamma) shifted past the row index,
    which consumes the generator exactly like rng.choice(concat(arange(i), arange(i+1, n)))
    and yields the same values (pinned in tests/test_host.py against the reference)."""
    rng = np.random.default_rng(seed)
    ids = rng.integers(0, n - 1, size=(n, gamma), dtype=np.int64)
    ids += ids >= np.arange(n)[:, None]
    srt = np.sort(ids, axis=1)
    bad = np.nonzero(np.any(srt[:, 1:] == srt[:, :-1], axis=1))[0]
    for i in bad:
        pick = rng.choice(n - 1, size=gamma, replace=False)
        ids[i] = pick + (pick >= i)
    return ids.astype(np.int32)


def restored_generator(seed: int, consumed32: int, buffered: int) -> np.random.Generator:
    """default_rng(seed) after `consumed32` 32-bit draws: PCG64 advanced past ceil(c / 2)
    outputs, with the unused high half of the last one buffered when c is odd (NumPy's
    has_uint32 / uinteger)."""
    rng = np.random.default_rng(seed)
    rng.bit_generator.advance((consumed32 + 1) // 2)
    if consumed32 % 2:
        st = rng.bit_generator.state
        st["has_uint32"] = 1
        st["uinteger"] = int(buffered)
        rng.bit_generator.state = st
    return rng


def init_random_rows_device(dev: DeviceIndex, n: int, gamma: int, seed: int) -> None:
    """init_random_ids with the bulk draw on the device (bit-identical): the device fills the
    rows and reports how many PCG64 outputs it consumed; rows with a repeated id are redrawn
    here from the same generator advanced past those outputs, in ascending row order."""
    consumed32, buffered, bad = dev.init_random_ids(seed)
    if bad.size:
        rng = restored_generator(seed, consumed32, buffered)
        rows = np.empty((bad.size, gamma), np.int32)
        for j, i in enumerate(bad):
            pick = rng.choice(n - 1, size=gamma, replace=False)
            rows[j] = pick + (pick >= i)
        dev.set_rows(bad, rows)


def _quality_sample(n: int, params: BuildParams) -> np.ndarray:
    rng = np.random.default_rng(params.seed + 1)
    size = min(params.quality_sample, n)
    return np.sort(rng.choice(n, size=size, replace=False)).astype(np.int64)


def _psi(dev: DeviceIndex, quality: QualityEstimate) -> float:
    """graph_quality (_kernels.py:207-224): GPU rows, host sum in the reference's order."""
    rows, counts = dev.get_rows(quality.sample_ids)
    gt = quality.ground_truth
    k = gt.shape[1]
    total = 0.0
    for si in range(gt.shape[0]):
        c = min(k, int(counts[si]))
        hits = int(np.isin(rows[si, :c], gt[si]).sum())
        total += hits / k
    return total / gt.shape[0]


def init_random_graph(features, attrs, schema, params: BuildParams, metric: MetricConfig,
                      _pull: bool = True) -> RelationGraph:
    features = np.ascontiguousarray(features, dtype=np.float32)
    attrs = np.ascontiguousarray(attrs, dtype=np.int32)
    n = features.shape[0]
    g = params.gamma
    if n <= g:
        raise ValueError(f"dataset size {n} must exceed gamma {g}; use a smaller gamma")
    dev = DeviceIndex(features, attrs, g)
    init_random_rows_device(dev, n, g, params.seed)
    dev.init_graph(None, 1.0 / metric.alpha)
    ids = np.empty((n, g), np.int32)  # filled by _pull
    graph = RelationGraph(features=features, attrs=attrs, schema=schema, metric=metric,
                          sigma=params.sigma, nbr_ids=ids, nbr_dists=np.empty((n, g), np.float32),
                          nbr_counts=np.full(n, g, np.int32), nbr_flags=np.ones((n, g), np.uint8),
                          _device=dev, _dev_sync=True)
    if _pull:
        graph._pull()
    return graph


def prepare_quality_estimate(graph: RelationGraph, params: BuildParams) -> QualityEstimate:
    k = params.quality_k or params.gamma
    sample = _quality_sample(graph.n, params)
    gt = graph.device().bf_topk_nodes(sample, k, 1.0 / graph.metric.alpha)
    return QualityEstimate(sample_ids=sample, ground_truth=gt)


def estimate_graph_quality(graph: RelationGraph, quality: QualityEstimate) -> float:
    psi = _psi(graph.device(), quality)
    quality.psi = psi
    return psi


def descent_iteration(graph: RelationGraph, params: BuildParams, _pull: bool = True) -> int:
    if graph.frozen:
        raise ValueError("graph is frozen")
    if graph.nbr_flags is None:
        raise ValueError("graph has no build flags (already pruned?)")
    inserted, pairs = graph.device().descent_iteration(params.gamma_new, 1.0 / graph.metric.alpha)
    graph.build_log.setdefault("pairs", []).append(pairs)
    if _pull:
        graph._pull()
    else:
        graph._dev_sync = True  # device is authoritative until the next pull
    return int(inserted)


def run_descent(features, attrs, schema, params: BuildParams, metric: MetricConfig,
                _pull: bool = True) -> RelationGraph:
    """_pull=False (build()): the rows stay on the device for semantic_prune; the host arrays
    are refreshed by its download."""
    t0 = time.perf_counter()
    graph = init_random_graph(features, attrs, schema, params, metric, _pull=False)
    t_init = time.perf_counter() - t0
    quality = prepare_quality_estimate(graph, params)
    graph.quality = quality
    psi_history = [estimate_graph_quality(graph, quality)]
    termination = "quality_reached"
    iterations = 0
    t_iter = []
    while psi_history[-1] < params.psi_target:
        if iterations >= params.max_iterations:
            termination = "max_iterations"
            break
        t1 = time.perf_counter()
        changes = descent_iteration(graph, params, _pull=False)
        iterations += 1
        psi_history.append(estimate_graph_quality(graph, quality))
        t_iter.append(time.perf_counter() - t1)
        if changes == 0:
            if psi_history[-1] < params.psi_target:
                termination = "converged_below_target"
            break
    if _pull:
        graph._pull()
    graph.build_log.update({
        "iterations": iterations,
        "psi_history": psi_history,
        "psi": psi_history[-1],
        "termination": termination,
        "seconds_init": t_init,
        "seconds_iterations": t_iter,
    })
    return graph


def semantic_prune(graph: RelationGraph, params: BuildParams) -> RelationGraph:
    """Prune, reinforce and reconnect (graph.py:202-232) on the device."""
    if graph.frozen:
        raise ValueError("graph is frozen")
    t0 = time.perf_counter()
    dev = graph.device()
    rounds = dev.prune(params.sigma)
    overflow, sweeps = dev.reinforce(params.sigma)
    graph.nbr_flags = None
    graph._pull()
    graph.build_log.update({"prune_guard_rounds": rounds, "reinforce_overflow_rows": overflow,
                            "reconnect_sweeps": sweeps,
                            "seconds_prune": time.perf_counter() - t0})
    return graph


def build(features, attrs, schema, params: BuildParams, metric: MetricConfig) -> RelationGraph:
    t0 = time.perf_counter()
    graph = run_descent(features, attrs, schema, params, metric, _pull=False)
    semantic_prune(graph, params)
    graph.frozen = True
    # the search-ready layout (locality order, u8 copy) is part of the build
    t1 = time.perf_counter()
    graph.device().route_prepare()
    graph.build_log["seconds_route_layout"] = time.perf_counter() - t1
    graph.build_log["seconds_total"] = time.perf_counter() - t0
    return graph


# ---------------------------------------------------------------------------
# "HELP" v1 index: magic, <IQIII header, <dBBddIqQI metric provenance, <d sigma, UTF-8
# dictionaries, f32 features, u32 attrs, then per node u32 count, count x u32 ids,
# count x f32 dists (the ids block precedes the dists block).
def write_index(graph: RelationGraph, path) -> None:
    n, m = graph.features.shape
    l = graph.attrs.shape[1]
    st = graph.metric.stats
    out = [INDEX_MAGIC, struct.pack("<IQIII", INDEX_VERSION, n, m, l, graph.gamma),
           struct.pack("<dBBddIqQI", graph.metric.alpha, int(bool(graph.metric.override)),
                       int(st is not None), st.avg_feature_distance if st else 0.0,
                       st.avg_attribute_distance if st else 0.0, st.sample_size if st else 0,
                       st.rng_seed if st else 0, graph.metric.n_total, graph.metric.l_dims),
           struct.pack("<d", graph.sigma)]
    for words in graph.schema.dictionaries:
        out.append(struct.pack("<I", len(words)))
        for w in words:
            b = w.encode("utf-8")
            out.append(struct.pack("<I", len(b)) + b)
    out.append(np.ascontiguousarray(graph.features, "<f4").tobytes())
    out.append(np.ascontiguousarray(graph.attrs, "<u4").tobytes())
    counts = np.asarray(graph.nbr_counts)
    for i in range(n):
        c = int(counts[i])
        out.append(struct.pack("<I", c))
        out.append(np.ascontiguousarray(graph.nbr_ids[i, :c], "<u4").tobytes())
        out.append(np.ascontiguousarray(graph.nbr_dists[i, :c], "<f4").tobytes())
    with open(path, "wb") as f:
        f.write(b"".join(out))


def read_index(path) -> RelationGraph:
    buf = open(path, "rb").read()
    pos = 0

    def need(size):
        if pos + size > len(buf):
            raise FormatError(f"{path}: truncated index file", offset=pos)

    def take(fmt):
        nonlocal pos
        size = struct.calcsize(fmt)
        need(size)
        vals = struct.unpack_from(fmt, buf, pos)
        pos += size
        return vals

    def take_array(dtype, count):
        nonlocal pos
        dt = np.dtype(dtype)
        need(dt.itemsize * count)
        a = np.frombuffer(buf, dtype=dt, count=count, offset=pos)
        pos += dt.itemsize * count
        return a

    if buf[:4] != INDEX_MAGIC:
        raise FormatError(f"{path}: bad magic", offset=0)
    pos = 4
    version, n, m, l, gamma = take("<IQIII")
    if version != INDEX_VERSION:
        raise FormatError(f"{path}: unsupported index version {version}", offset=4)
    alpha, override, has_stats, s_v, s_a, ssize, sseed, n_total, l_dims = take("<dBBddIqQI")
    (sigma,) = take("<d")
    dicts = []
    for _ in range(l):
        (cnt,) = take("<I")
        words = []
        for _ in range(cnt):
            (wl,) = take("<I")
            need(wl)
            words.append(buf[pos:pos + wl].decode("utf-8"))
            pos += wl
        dicts.append(tuple(words))
    features = take_array("<f4", n * m).reshape(n, m).astype(np.float32)
    attrs = take_array("<u4", n * l).reshape(n, l).astype(np.int32)
    ids = np.zeros((n, gamma), np.int32)
    dists = np.full((n, gamma), np.inf, np.float32)
    counts = np.zeros(n, np.int32)
    for i in range(n):
        (c,) = take("<I")
        if c > gamma:
            raise FormatError(f"{path}: node {i} degree {c} exceeds capacity {gamma}", offset=pos - 4)
        ids[i, :c] = take_array("<u4", c)
        dists[i, :c] = take_array("<f4", c)
        counts[i] = c
    if pos != len(buf):
        raise FormatError(f"{path}: trailing bytes after adjacency block", offset=pos)
    stats = SampleStats(s_v, s_a, int(ssize), int(sseed)) if has_stats else None
    metric = MetricConfig(alpha=alpha, stats=stats, n_total=int(n_total), l_dims=int(l_dims),
                          override=bool(override))
    return RelationGraph(features=features, attrs=attrs, schema=AttributeSchema(tuple(dicts)),
                         metric=metric, sigma=sigma, nbr_ids=ids, nbr_dists=dists,
                         nbr_counts=counts, frozen=True)

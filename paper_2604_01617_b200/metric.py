"""AUTO metric definition and alpha calibration (host side).

U = S_V * (1 + S_A / alpha)  (reference metric.py:161-168).  alpha is
computed once on the host from sampled all-pairs means and handed to the kernels as
inv_alpha = 1 / alpha, exactly as the reference does (graph.py:131, router.py:84).
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np

from .errors import CalibrationError


@dataclass(frozen=True)
class AttributeSchema:
    """Per-dimension label dictionaries (reference dataset_io.py:30-58)."""

    dictionaries: tuple

    @property
    def l(self) -> int:
        return len(self.dictionaries)

    @property
    def cardinalities(self) -> tuple:
        return tuple(len(d) for d in self.dictionaries)


@dataclass(frozen=True)
class SampleStats:
    """Sampled mean feature / attribute distances (reference dataset_io.py:61-74)."""

    avg_feature_distance: float
    avg_attribute_distance: float
    sample_size: int
    rng_seed: int


@dataclass(frozen=True)
class MetricConfig:
    """Fused-distance configuration (reference metric.py:25-44)."""

    alpha: float
    stats: SampleStats | None
    n_total: int
    l_dims: int
    override: bool = False

    def __post_init__(self):
        if self.alpha <= 0:
            raise ValueError("alpha must be positive")
        if self.l_dims < 1:
            raise ValueError("l_dims must be >= 1")

    @classmethod
    def manual(cls, alpha: float, l_dims: int, n_total: int = 0) -> "MetricConfig":
        return cls(alpha=alpha, stats=None, n_total=n_total, l_dims=l_dims, override=True)


def sample_statistics(features, attributes, sample_size: int, seed: int = 0) -> SampleStats:
    """All-pairs means over a NumPy-drawn sample (reference dataset_io.py:247-267).

    Kept on the host with SciPy's pdist so alpha is bit-identical to the reference's."""
    from scipy.spatial.distance import pdist

    features = np.asarray(features)
    attributes = np.asarray(attributes)
    n = features.shape[0]
    if sample_size < 2:
        raise ValueError("sample_size must be >= 2")
    if sample_size > n:
        raise ValueError("sample_size exceeds dataset size")
    pick = np.random.default_rng(seed).choice(n, size=sample_size, replace=False)
    s_v = float(pdist(features[pick].astype(np.float64), metric="euclidean").mean())
    s_a = float(pdist(attributes[pick].astype(np.float64), metric="cityblock").mean())
    return SampleStats(s_v, s_a, sample_size, seed)


def norm_scale(x: float) -> float:
    """Decade shift into (0.1, 1] (reference metric.py:110-125)."""
    if x < 0:
        raise ValueError("norm_scale requires a non-negative input")
    if x == 0:
        raise ValueError("norm_scale is undefined at 0")
    while x > 1.0:
        x /= 10.0
    while x <= 0.1:
        x *= 10.0
    return x


def compute_alpha(stats: SampleStats, n_total: int, l_dims: int) -> MetricConfig:
    """alpha = Norm(N / S_V) + Norm(S_A / L) (reference metric.py:128-158)."""
    if n_total < 1:
        raise ValueError("n_total must be >= 1")
    if l_dims < 1:
        raise ValueError("l_dims must be >= 1")
    if stats.avg_feature_distance == 0:
        raise CalibrationError("degenerate feature space: mean sampled feature distance is 0")
    term_v = norm_scale(n_total / stats.avg_feature_distance)
    if stats.avg_attribute_distance == 0:
        warnings.warn("mean sampled attribute distance is 0; attribute term of alpha set to 0",
                      stacklevel=2)
        term_a = 0.0
    else:
        term_a = norm_scale(stats.avg_attribute_distance / l_dims)
    return MetricConfig(alpha=term_v + term_a, stats=stats, n_total=n_total, l_dims=l_dims)


def fused_distance(node_feature, node_attrs, query_feature, query_attrs, config: MetricConfig,
                   mask=None) -> float:
    """Scalar AUTO distance of one node against one query (reference metric.py:161-168)."""
    d = np.asarray(node_feature, np.float64) - np.asarray(query_feature, np.float64)
    s_v = float(np.sqrt(np.sum(d * d)))
    a = np.abs(np.asarray(node_attrs, np.int64) - np.asarray(query_attrs, np.int64))
    if mask is not None:
        a = a * np.asarray(mask, np.int64)
    return s_v * (1.0 + float(a.sum()) / config.alpha)

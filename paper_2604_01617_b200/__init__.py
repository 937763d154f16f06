"""STABLE hot path on B200 (sm_100a): the AUTO heterogeneous metric evaluated in bulk for
exhaustive top-k, HELP graph construction and Dynamic Heterogeneity Routing.

Drop-in for the reference package `hybridann` 0.1.0 on that path: same names, argument
meaning, return types and errors (reference __init__.py:62-109, hot-path subset).  Bulk work
runs in libstable_b200.so (hand-written CUDA behind the C ABI of include/stable_b200.h);
there is no CPU fallback.
"""

__version__ = "0.1.0"

from .errors import (CalibrationError, ConstraintError, FormatError, HybridAnnError,
                     MappingError)
from .evaluate import (CSV_FIELDS, ROOFLINE_FIELDS, SweepRow, bench_sweep, mean_recall,
                       oracle_auto_topk, oracle_auto_topk_batch, oracle_hybrid_groundtruth,
                       oracle_hybrid_groundtruth_batch, recall_at_k, write_sweep_csv)
from .graph import (BuildParams, QualityEstimate, RelationGraph, build, descent_iteration,
                    estimate_graph_quality, init_random_graph, init_random_ids,
                    prepare_quality_estimate, read_index, run_descent, semantic_prune,
                    write_index)
from .metric import (AttributeSchema, MetricConfig, SampleStats, compute_alpha, fused_distance,
                     norm_scale, sample_statistics)
from .router import (SearchParams, SearchStats, entry_points, search, search_batch,
                     search_batch_arrays)

__all__ = [
    "AttributeSchema", "BuildParams", "CalibrationError", "ConstraintError", "FormatError",
    "HybridAnnError", "MappingError", "MetricConfig", "QualityEstimate", "RelationGraph",
    "SampleStats", "SearchParams", "SearchStats", "SweepRow", "bench_sweep", "build",
    "compute_alpha", "descent_iteration", "entry_points", "estimate_graph_quality",
    "fused_distance", "init_random_graph", "init_random_ids", "mean_recall", "norm_scale",
    "oracle_auto_topk", "oracle_auto_topk_batch", "oracle_hybrid_groundtruth",
    "oracle_hybrid_groundtruth_batch", "CSV_FIELDS", "ROOFLINE_FIELDS",
    "prepare_quality_estimate", "read_index", "recall_at_k", "run_descent",
    "sample_statistics", "search", "search_batch", "search_batch_arrays", "semantic_prune",
    "write_index", "write_sweep_csv",
]

"""pytest plugin: run the REFERENCE's own test suite with its kernel module swapped for ours.

The reference resolves every hot-path kernel as ``_kernels.<fn>`` at call time
(graph.py:13, router.py:15), so replacing the module attributes routes its unmodified
orchestration (build, run_descent, semantic_prune, search, ...) through the B200 C ABI.
Loaded with ``-p swap_plugin`` from tests/test_ref_swap.py; prints one SWAP line per kernel so
the caller can check that every swapped kernel was really called.
"""

import collections

import os

import hybridann._kernels as _ref_kernels

if os.environ.get("SWAP_TARGET", "b200") == "oracle":
    # CPU check of the swap mechanics and of the oracle itself: the C restatement stands in
    from oracle.oracle import kernels as _gpu_kernels
    _gpu_kernels.__all__ = ["compute_row_distances", "build_candidates", "local_join",
                            "brute_force_topk", "graph_quality", "count_in_degrees",
                            "prune_pass", "reinforce_pass", "reconnect_islands", "route"]
else:
    import paper_2604_01617_b200._kernels as _gpu_kernels

CALLS = collections.Counter()


def _counted(name, fn):
    def wrapper(*args, **kwargs):
        CALLS[name] += 1
        return fn(*args, **kwargs)
    wrapper.__name__ = name
    return wrapper


for _name in _gpu_kernels.__all__:
    if not hasattr(_ref_kernels, _name):
        raise RuntimeError(f"reference _kernels has no {_name}")
    setattr(_ref_kernels, _name, _counted(_name, getattr(_gpu_kernels, _name)))


def pytest_terminal_summary(terminalreporter):
    terminalreporter.section("kernel swap")
    for name in _gpu_kernels.__all__:
        terminalreporter.write_line(f"SWAP {name} calls={CALLS[name]}")

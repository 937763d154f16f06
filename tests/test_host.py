"""CPU tests of the product's host side: the C-ABI library loads and exports every symbol
the header declares, the entry-point RNG port equals NumPy (and the reference's vectors),
and the host init-id draw equals the reference's."""

import os
import re

import numpy as np
import pytest

import paper_2604_01617_b200 as sb
from paper_2604_01617_b200 import _lib
from paper_2604_01617_b200.device import entry_points_host

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    header = open(os.path.join(ROOT, "include", "stable_b200.h")).read()
    declared = set(re.findall(r"\b(sb_[a-z0-9_]+)\s*\(", header))
    assert declared, "header declares no entry points"
    lib = _lib.load()
    for name in sorted(declared):
        assert hasattr(lib, name), f"{name} declared in stable_b200.h but not exported"
    assert declared == set(_lib.exported_symbols()), "ctypes table out of sync with the header"
    assert lib.sb_version() == 1


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_errors_map_to_reference_types():
    with pytest.raises(ValueError):
        _lib.call("sb_entry_points", 10, 0, 0, 0, 1, None)


def test_entry_points_match_reference_vectors(rng_golden):
    gd = rng_golden
    seen = 0
    for key in gd.files:
        if key.startswith("ep_"):
            _, n, k, seed, qi = key.split("_")
            got = entry_points_host(int(n), int(k), int(seed), int(qi), 1)[0]
            np.testing.assert_array_equal(got, gd[key], err_msg=key)
            seen += 1
        elif key.startswith("ephead_"):
            _, n, k, seed, qi = key.split("_")
            got = entry_points_host(int(n), int(k), int(seed), int(qi), 1)[0]
            np.testing.assert_array_equal(got[:256], gd[key], err_msg=key)
            import hashlib
            a = np.ascontiguousarray(got)
            h = hashlib.sha256(a.tobytes() + str(a.dtype).encode() + str(a.shape).encode()).hexdigest()
            assert h == str(gd[f"epsha_{n}_{k}_{seed}_{qi}"]), key
            seen += 1
    assert seen >= 40


@pytest.mark.parametrize("n,k", [(2, 1), (2, 2), (17, 17), (9999, 200), (10000, 10000),
                                 (10001, 200), (10001, 201), (50000, 1000), (50000, 1001),
                                 (123457, 64), (2000000, 40001)])
def test_entry_points_match_numpy(n, k):
    for seed, qi in ((0, 0), (1, 5), (7, 123456), (2**40 + 3, 2**33 + 1)):
        want = np.random.default_rng(np.random.SeedSequence(entropy=(seed, qi))).choice(
            n, size=k, replace=False)
        got = entry_points_host(n, k, seed, qi, 1)[0]
        np.testing.assert_array_equal(got, want)


def test_entry_points_batch_is_per_query_stream():
    got = entry_points_host(5000, 30, 3, 10, 4)
    for r in range(4):
        want = np.random.default_rng(np.random.SeedSequence(entropy=(3, 10 + r))).choice(
            5000, size=30, replace=False)
        np.testing.assert_array_equal(got[r], want)
    np.testing.assert_array_equal(sb.entry_points(5000, 30, 3, 11), got[1])


def test_init_ids_match_reference(rng_golden):
    gd = rng_golden
    import hashlib
    for key in gd.files:
        if not key.startswith("initsha_"):
            continue
        _, n, g, seed = key.split("_")
        ids = sb.init_random_ids(int(n), int(g), int(seed))
        h = hashlib.sha256(ids.tobytes() + str(ids.dtype).encode() + str(ids.shape).encode()).hexdigest()
        assert h == str(gd[key]), key
        full = f"init_{n}_{g}_{seed}"
        if full in gd.files:
            np.testing.assert_array_equal(ids, gd[full])
        assert len(gd[f"initbad_{n}_{g}_{seed}"]) >= 0


def test_init_ids_resample_path_exercised(rng_golden):
    # at least one fixture must contain duplicate-row resamples
    assert any(len(rng_golden[k]) > 0 for k in rng_golden.files if k.startswith("initbad_"))


def test_alpha_host_matches_reference(small_golden):
    gd = small_golden
    st = sb.sample_statistics(gd["features"], gd["attrs"], 300, seed=13)
    cfg = sb.compute_alpha(st, 600, 3)
    assert cfg.alpha == float(gd["alpha"])


def test_build_params_validation():
    with pytest.raises(ValueError):
        sb.BuildParams(gamma=1)
    with pytest.raises(ValueError):
        sb.BuildParams(sigma=1.5)
    with pytest.raises(ValueError):
        sb.BuildParams(psi_target=2.0)


def test_pioneer_default_and_validation():
    assert sb.SearchParams(k=20).resolved_pioneer_size() == 10
    assert sb.SearchParams(k=1).resolved_pioneer_size() == 1
    with pytest.raises(ValueError):
        sb.SearchParams(k=20, pioneer_size=21).resolved_pioneer_size()


def test_recall_at_k_semantics():
    assert sb.recall_at_k([1, 2, 3], [1, 2, 3], 3) == 1.0
    assert sb.recall_at_k([5, 1, 7, 8, 9], [1, 5], 5) == 1.0
    assert sb.recall_at_k([7, 8], [], 2) == 1.0
    with pytest.raises(ValueError):
        sb.recall_at_k([1], [1], 0)


def test_index_format_round_trip_host(small_golden, tmp_path):
    gd = small_golden
    g = sb.RelationGraph(features=gd["features"], attrs=gd["attrs"],
                         schema=sb.AttributeSchema((("v1", "v2", "v3"),) * 3),
                         metric=sb.MetricConfig.manual(float(gd["alpha"]), 3), sigma=0.44,
                         nbr_ids=gd["final_ids"], nbr_dists=gd["final_dists"],
                         nbr_counts=gd["final_counts"], frozen=True)
    p1, p2 = tmp_path / "a.idx", tmp_path / "b.idx"
    sb.write_index(g, p1)
    g2 = sb.read_index(p1)
    sb.write_index(g2, p2)
    assert p1.read_bytes() == p2.read_bytes()
    np.testing.assert_array_equal(g2.nbr_counts, g.nbr_counts)
    for i in range(g.n):
        c = g.nbr_counts[i]
        np.testing.assert_array_equal(g2.nbr_ids[i, :c], g.nbr_ids[i, :c])
    p1.write_bytes(p1.read_bytes()[:-3])
    with pytest.raises(sb.FormatError, match="truncated"):
        sb.read_index(p1)


def test_no_cpu_fallback(tmp_path):
    """The product path has no CPU fallback: without a GPU every device entry point raises,
    and a missing shared library raises at load time."""
    import subprocess
    import sys
    from paper_2604_01617_b200 import _lib
    from paper_2604_01617_b200.device import DeviceIndex
    if _lib.device_count() == 0:
        with pytest.raises(RuntimeError, match="no CUDA device"):
            DeviceIndex(np.zeros((10, 4), np.float32), np.ones((10, 1), np.int32), 4)
    code = ("import paper_2604_01617_b200._lib as L\n"
            "try:\n    L.load()\nexcept RuntimeError as e:\n    print('raised', e)\n")
    env = dict(os.environ, STABLE_B200_LIB=str(tmp_path / "missing.so"))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert "raised" in out.stdout and "missing" in out.stdout


def test_index_file_written_by_reference():
    """tests/golden/small_index.help was written by the reference's own write_index
    (graph.py:287-330; tests/golden/make_golden.py case_index).  read_index gives the arrays
    the reference's read_index gave (stale tails as id 0 / +inf, graph.py:380-381), and
    write_index of that graph reproduces the file byte for byte."""
    import hashlib
    import tempfile
    path = os.path.join(os.path.dirname(__file__), "golden", "small_index.help")
    gd = np.load(os.path.join(os.path.dirname(__file__), "golden", "index.npz"))
    raw = open(path, "rb").read()
    assert hashlib.sha256(raw).hexdigest() == str(gd["file_sha"])
    g = sb.read_index(path)
    np.testing.assert_array_equal(g.nbr_counts, gd["counts"])
    np.testing.assert_array_equal(g.nbr_ids, gd["ids"])
    np.testing.assert_array_equal(g.nbr_dists, gd["dists"])
    assert g.frozen and g.gamma == 24 and g.n == 600
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "again.help")
        sb.write_index(g, out)
        assert open(out, "rb").read() == raw


def test_sweep_csv_matches_reference(tmp_path):
    """write_sweep_csv writes the reference's CSV byte for byte (evaluate.py:144-158; the
    reference's own output of the same rows is in tests/golden/index.npz); roofline=True
    appends exactly the two roofline columns."""
    gd = np.load(os.path.join(os.path.dirname(__file__), "golden", "index.npz"))
    rows = [sb.evaluate.SweepRow(k=10, pioneer=5, mean_recall_at_10=0.95123456, qps=1234.5678,
                                 mean_dist_evals=321.123, n_queries=20),
            sb.evaluate.SweepRow(k=200, pioneer=100, mean_recall_at_10=1.0, qps=7.0,
                                 mean_dist_evals=4152.84, n_queries=10000, algorithmic_gbs=3264.5,
                                 hbm_frac=0.5051)]
    p = tmp_path / "s.csv"
    sb.evaluate.write_sweep_csv(p, rows)
    assert p.read_text() == str(gd["sweep_csv"])
    sb.evaluate.write_sweep_csv(p, rows, roofline=True)
    lines = p.read_text().splitlines()
    assert lines[0] == ",".join(sb.evaluate.CSV_FIELDS + ["algorithmic_gbs", "hbm_frac"])
    assert lines[2].endswith(",3264.5,0.5051")

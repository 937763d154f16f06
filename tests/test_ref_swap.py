"""Drop-in proof at the kernel level: the reference's OWN test suite (hybridann 0.1.0,
/root/reference/pkg/tests, installed unmodified into the git-ignored baseline/_ref/ by
tools/install_ref.sh) run with ``hybridann._kernels`` swapped for
``paper_2604_01617_b200._kernels`` (tests/ref_swap/swap_plugin.py; on CPU the same run with
the oracle's C restatement swapped in pins the oracle with the reference's tests).  Every one of the
reference's tests must pass, every swapped kernel must have been called, and the acceptance
criteria must print the numbers the reference recorded on its own CPU run
(pkg/test_output.txt:105-115).  Skips (never passes silently) when baseline/_ref is absent.
"""

import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

# the reference's recorded acceptance numbers (pkg/test_output.txt:105-115): criterion ->
# substrings its detail must contain (timings excluded)
RECORDED = {
    1: ["alpha=0.742911"],
    2: ["530712 mismatched pairs, 0 violations"],
    3: ["10000 tuples, 0 disagreements"],
    4: ["all clean"],
    5: ["psi=0.9409 after 2 iterations"],
    6: ["fused=1.0000 exact=1.0000"],
    7: ["recall=1.0000"],
    8: ["coarse+refine=2197.6 refine-only=2202.2"],
    9: ["100/100 queries exact"],
    10: ["bit_exact=True search_identical=True"],
    11: ["sigma=0.4:1.0000 sigma=0.44:1.0000 sigma=0.5:1.0000 spread=0.00000"],
}


def _need_ref():
    if not os.path.isdir(os.path.join(REF, "site", "hybridann")):
        pytest.skip("baseline/_ref not installed (run tools/install_ref.sh where /root/reference "
                    "exists); the reference-suite swap test cannot run")


def _run_reference_suite(target):
    _need_ref()
    env = dict(os.environ)
    env["SWAP_TARGET"] = target
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(REF, "site"), ROOT,
                                         os.path.join(ROOT, "tests", "ref_swap"),
                                         env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "tests", "-q", "-p", "swap_plugin",
           "-p", "no:cacheprovider", "-o", "addopts=", "--rootdir", REF]
    r = subprocess.run(cmd, cwd=REF, env=env, capture_output=True, text=True, timeout=3000)
    out = r.stdout + r.stderr
    tail = out[-6000:]
    assert r.returncode == 0, tail
    m = re.search(r"(\d+) passed", out)
    assert m and int(m.group(1)) == 86 and " failed" not in out, tail
    calls = dict(re.findall(r"SWAP (\w+) calls=(\d+)", out))
    assert len(calls) == 10, tail
    for name, c in calls.items():
        assert int(c) > 0, f"swapped kernel {name} never called\n{tail}"
    crit = {int(k): v for k, v in re.findall(r"CRITERION\s+(\d+) \[PASS\] (.*)", out)}
    assert sorted(crit) == list(range(1, 12)), tail
    for num, needles in RECORDED.items():
        for needle in needles:
            assert needle in crit[num], f"criterion {num}: {crit[num]!r} lacks {needle!r}"


@pytest.mark.gpu
def test_reference_suite_with_b200_kernels():
    _run_reference_suite("b200")


def test_reference_suite_with_oracle_kernels():
    _run_reference_suite("oracle")

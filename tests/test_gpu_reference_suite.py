"""The reference's own hot-path tests, unchanged, on the B200 through the
drop-in (SURVEY.md 7.1 test plan item 1): /root/reference/pkg/tests/test_accel.py
(all of it) and test_acceptance.py criteria 1, 8, 9, 10, with mintri.accel's
query functions routed to paper_2112_05570_b200.accel by
tests/reference_suite/mwt_dropin_plugin.py.

The unmodified reference package and those test files come from
baseline/_ref (tools/install_reference.sh; git-ignored, shipped to the GPU box).
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "reference_tests")

pytestmark = pytest.mark.gpu

SELECTION = ["test_accel.py",
             "test_acceptance.py::test_criterion_01_oracle_equivalence",
             "test_acceptance.py::test_criterion_08_grass_decreasing_traversal",
             "test_acceptance.py::test_criterion_09_bvh_logn_trend",
             "test_acceptance.py::test_criterion_10_kd_diagonal_pathology"]


def test_reference_accel_and_acceptance_tests_through_the_drop_in():
    if not (os.path.isdir(os.path.join(REF, "mintri")) and os.path.isdir(REF_TESTS)):
        pytest.skip("reference not installed in baseline/_ref (tools/install_reference.sh)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, ROOT, os.path.join(ROOT, "tests", "reference_suite"), REF_TESTS,
                                         env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "mwt_dropin_plugin", "-p", "no:cacheprovider",
           "--rootdir", REF_TESTS, "-o", "addopts=", "-s"] + SELECTION
    r = subprocess.run(cmd, cwd=REF_TESTS, env=env, capture_output=True, text=True, timeout=3000)
    out = r.stdout + r.stderr
    log = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(log):
        with open(os.path.join(log, "reference_suite.log"), "w") as fh:
            fh.write(out)
    assert r.returncode == 0, out[-6000:]
    assert "mwt drop-in:" in out
    # the reference tests really went through the drop-ins
    line = [ln for ln in out.splitlines() if ln.startswith("mwt drop-in calls:")][-1]
    calls = dict(kv.split("=") for kv in line.split(":", 1)[1].strip().split(", "))
    for q in ("traverse_triangulation", "bvh_intersect", "kd_intersect"):
        assert int(calls[q]) > 0, line
    for c in ("criterion 1", "criterion 8", "criterion 9", "criterion 10"):
        assert f"PASS {c}:" in out, c

"""The reference's own test suite (pkg/tests, 228 tests) run against the drop-in, through both seams.

The reference package and its tests are staged -- unmodified, never committed -- into
``baseline/_ref`` by ``tools/stage_reference.sh`` (the driver's reference-install directory, which
travels to the GPU box).  ``QUBRUTE_REF`` overrides the location.  Each run copies the tests to a
temporary directory and runs them in a fresh interpreter with ``tests/refsuite/qb_seam_plugin.py``,
which reroutes the hot path to libqubrute_b200.so before collection:

* seam 1   -- ``qubrute._kernels.gray_scan`` (SURVEY.md §8b Seam 1);
* seam 2   -- ``solve_incremental`` / ``solve_parallel`` / ``solve_subspace`` with the reference's own
              ``QuboInstance`` / ``SolveConfig`` objects (Seam 2);
* seam 2full -- Seam 2 plus ``solve_naive`` / ``solve`` and INTEGRATION.md's CLI recipe
              (``qubrute.cli.solve = b2.solve``); criterion 6 (naive-vs-Gray speed-up) is skipped
              with its reason, every other test must pass.

The CPU test below checks the seam-2 boundary types without a GPU (the reference's ``SolveConfig``
reaches the backend instead of failing in Python).
"""

import os
import re
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
REF = os.environ.get("QUBRUTE_REF") or os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "qubrute_tests")
HAVE_REF = os.path.isdir(os.path.join(REF, "qubrute")) and os.path.isdir(REF_TESTS)
needs_ref = pytest.mark.skipif(not HAVE_REF, reason=f"reference not staged at {REF} (run tools/stage_reference.sh)")


def _ref_env():
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, os.path.join(ROOT, "tests", "refsuite"), ROOT,
                                         env.get("PYTHONPATH", "")])
    env["QB_REPO_ROOT"] = ROOT
    return env


@needs_ref
def test_reference_solveconfig_reaches_backend():
    """Seam 2 boundary on CPU: the reference's SolveConfig / QuboInstance pass the drop-in's Python
    layer (the round-1 AttributeError on ``config.devices``) and stop only at the missing GPU."""
    code = r"""
import numpy as np, qubrute, paper_2310_19373_b200 as b2
from paper_2310_19373_b200._lib import BackendError
inst = qubrute.random_instance(8, seed=3)
for call in (lambda: b2.solve_parallel(inst, qubrute.SolveConfig(threads=4)),
             lambda: b2.solve(inst, qubrute.SolveConfig(threads=4, mode="parallel")),
             lambda: b2.solve(inst, qubrute.SolveConfig(mode="incremental"))):
    try:
        call()
        print("ran")
    except BackendError:
        print("backend")
try:
    b2.solve_parallel(inst, qubrute.SolveConfig(threads=1, fixed_bits=8))
except ValueError as e:
    print("valueerror", e)
big = qubrute.QuboInstance(np.zeros((41, 41)), max_n=41)
for call in (lambda: b2.solve_incremental(big), lambda: b2.solve_naive(qubrute.random_instance(10, seed=1), max_n=8)):
    try:
        call()
    except qubrute.DimensionCapError as e:
        assert isinstance(e, b2.DimensionCapError)
        print("caperror")
"""
    r = subprocess.run([sys.executable, "-c", code], env=_ref_env(), capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.split()
    assert "AttributeError" not in r.stderr
    assert lines.count("ran") + lines.count("backend") == 3, r.stdout
    assert "valueerror" in r.stdout
    assert lines.count("caperror") == 2, r.stdout  # reference-typed cap errors (test_solver.py:55-58,102-105)


def _run_suite(seam: str, tmp_path):
    dst = tmp_path / "qubrute_tests"
    shutil.copytree(REF_TESTS, dst)
    env = _ref_env()
    env["QB_SEAM"] = seam
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "qb_seam_plugin", "-p", "no:cacheprovider",
                        "-rs", str(dst)], cwd=str(tmp_path), env=env, capture_output=True, text=True, timeout=3000)
    log = r.stdout + "\n" + r.stderr
    out_dir = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out_dir):
        with open(os.path.join(out_dir, f"refsuite_seam{seam}.log"), "w") as fh:
            fh.write(log)
    return r.returncode, log


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("seam", ["1", "2", "2full"])
def test_reference_suite_through_seam(seam, tmp_path):
    rc, log = _run_suite(seam, tmp_path)
    assert rc == 0, log[-6000:]
    passed = int(re.search(r"(\d+) passed", log).group(1))
    m = re.search(r"b200_calls=(\d+)", log)
    assert m and int(m.group(1)) > 0, "the B200 library was never called"
    skipped = re.findall(r"SKIPPED \[\d+\] (.*)", log)
    if seam == "2full":
        assert passed >= 227 and len(skipped) == 1 and "criterion 6" in skipped[0], log[-3000:]
    else:
        assert passed == 228 and not skipped, log[-3000:]

"""The reference's OWN tests, run against the B200 backends.

The reference package is staged (git-ignored) under baseline/_ref/pkg by
tools/stage_reference_suite.py, which `__graft_entry__.build()` runs.  Each
test below launches pytest on the reference's test files with
tests/refsuite_plugin.py, which registers the backends "cuda" (sweep-level
module protocol, bit-exact GPU sweeps) and "cuda-fit" (the device-resident
fit behind the reference's `pcd_fit`):

* /root/reference/pkg/tests/test_solver.py -- every `backend`-parametrised
  test (conftest.py:14-17) runs on compiled, python, cuda and cuda-fit,
  including worker invariance (:222-230), PCD == serialised round order
  (:203-219) and backends agreeing at convergence (:233-243);
* /root/reference/pkg/tests/test_acceptance.py criteria 04, 05, 06, 07, 10
  (:112-183, :216-225) with PARCONCORD_BACKEND set to each GPU backend, so
  the module-scoped fits themselves run on the GPU.
"""

import os
import re
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(REPO, "baseline", "_ref", "pkg")

pytestmark = pytest.mark.gpu


def _run(args, env_extra=None, timeout=1200):
    if not os.path.isdir(os.path.join(PKG, "tests")):
        pytest.skip("reference suite not staged (baseline/_ref/pkg): tools/stage_reference_suite.py, which "
                    "__graft_entry__.build() runs where /root/reference exists, stages it for the GPU box")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(PKG, "src"), os.path.join(PKG, "tests"),
                                         os.path.join(REPO, "tests"), REPO])
    env.pop("PARCONCORD_BACKEND", None)
    env.update(env_extra or {})
    cmd = [sys.executable, "-m", "pytest", "-p", "refsuite_plugin", "-p", "no:cacheprovider", "-q", "-rA",
           "--rootdir", PKG, *args]
    res = subprocess.run(cmd, cwd=PKG, env=env, capture_output=True, text=True, timeout=timeout)
    out = res.stdout + res.stderr
    sys.stdout.write(out[-6000:])
    return res.returncode, out


def _passed(out, pattern):
    return [line for line in out.splitlines() if line.startswith("PASSED") and re.search(pattern, line)]


def test_reference_solver_suite_on_cuda_backends():
    rc, out = _run(["tests/test_solver.py"])
    assert rc == 0, out[-4000:]
    cuda = _passed(out, r"\[cuda\]")
    fit = _passed(out, r"\[cuda-fit\]")
    # every backend-parametrised test of test_solver.py ran on both GPU backends
    assert len(cuda) >= 10 and len(fit) == len(cuda), (len(cuda), len(fit))
    assert _passed(out, r"test_backends_agree_at_convergence")


@pytest.mark.parametrize("backend", ["cuda", "cuda-fit"])
def test_reference_acceptance_criteria_on_cuda(backend):
    sel = "criterion_04 or criterion_05 or criterion_06 or criterion_07 or criterion_10"
    rc, out = _run(["tests/test_acceptance.py", "-s", "-k", sel], {"PARCONCORD_BACKEND": backend})
    assert rc == 0, out[-4000:]
    for num in ("04", "05", "06", "07", "10"):
        assert f"[criterion {num}] PASS" in out, num

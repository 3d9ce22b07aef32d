"""Stage the reference package's own test suite for a GPU run (test infrastructure).

    python tools/stage_reference_suite.py

Copies /root/reference/pkg to baseline/_ref/pkg and builds its compiled
backend there (the recipe of SURVEY.md 8c: `setup.py build_ext --inplace` with
/usr/bin/gcc).  baseline/_ref/ is git-ignored (the reference's sources never
enter this repo's history) but not gpurun-ignored, so it travels to the GPU
box, where tests/test_gpu_reference_suite.py runs the reference's
tests/test_solver.py and tests/test_acceptance.py with the B200 backends
registered by tests/refsuite_plugin.py.  `__graft_entry__.build()` calls this
whenever /root/reference exists.
"""

import os
import shutil
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "/root/reference/pkg"
DST = os.path.join(REPO, "baseline", "_ref", "pkg")


def stage(force=False):
    if not os.path.isdir(SRC):
        return None
    stamp = os.path.join(DST, ".staged")
    if os.path.exists(stamp) and not force:
        return DST
    if os.path.isdir(DST):
        shutil.rmtree(DST)
    shutil.copytree(SRC, DST, ignore=shutil.ignore_patterns("build", "*.so", "__pycache__", "*.egg-info"))
    subprocess.run(["chmod", "-R", "u+w", DST], check=True)
    env = dict(os.environ, CC="/usr/bin/gcc", LDSHARED="/usr/bin/gcc -shared")
    subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=DST, env=env, check=True,
                   capture_output=True)
    shutil.rmtree(os.path.join(DST, "build"), ignore_errors=True)
    open(stamp, "w").close()
    return DST


if __name__ == "__main__":
    print(stage(force="--force" in sys.argv))

"""pytest plugin: run the REFERENCE's own test suite against the B200 backends.

Loaded with `-p refsuite_plugin` by tests/test_gpu_reference_suite.py, with the
reference package staged under baseline/_ref/pkg (tools/stage_reference_suite.py)
first on PYTHONPATH.  It is the registration a maintainer would add to the
reference's `_backend.py`, applied as a monkeypatch so the
reference's sources stay untouched:

* backend "cuda"     -- the sweep-level module protocol (`_backend.py:36-49`,
  `_ckernels.pyx:53,68-70,105-106`): the reference's own `pcd_fit`/`cd_fit`
  loops (`solver.py:227-294`) call `paper_2106_09382_b200.cuda_kernels`, whose
  sweeps are bit-exact GPU kernels (csrc/pcd_exact.cu).
* backend "cuda-fit" -- the fit-level drop-in: the reference's `pcd_fit`
  dispatches to this repo's device-resident fit (one persistent kernel per
  fit, `Solver.fit` -> `concord_solver_fit`), with the reference's types and
  exceptions on both sides of the call.  `cd_fit` and custom schedules under
  this name use the sweep-level module, as this repo's own `pcd_fit` does.

The reference's `backend` fixture (`tests/conftest.py:14-17`) iterates
`available_backends()`, so every parametrised test runs on both names, and
`PARCONCORD_BACKEND=cuda|cuda-fit` makes them the default for the tests that
take no backend argument (test_acceptance.py).
"""

import os

import parconcord as ref
from parconcord import _backend as ref_backend
from parconcord import solver as ref_solver

import paper_2106_09382_b200 as ours
from paper_2106_09382_b200 import cuda_kernels

CUDA_NAMES = ("cuda", "cuda-fit")

_orig_available = ref_backend.available_backends
_orig_default = ref_backend.default_backend_name
_orig_get = ref_backend.get_backend
_orig_pcd_fit = ref_solver.pcd_fit


def available_backends():
    return tuple(_orig_available()) + CUDA_NAMES


def default_backend_name():
    env = os.environ.get("PARCONCORD_BACKEND")
    if env in CUDA_NAMES:
        return env
    return _orig_default()


def get_backend(name=None):
    if name is None:
        name = default_backend_name()
    if name in CUDA_NAMES:
        return cuda_kernels
    return _orig_get(name)


def _to_ref(rep):
    return ref_solver.FitReport(
        estimate=ref.PrecisionEstimate(rep.estimate.omega),
        iterations=rep.iterations,
        final_delta=rep.final_delta,
        converged=rep.converged,
        objective_trace=tuple(rep.objective_trace),
        edge_count=rep.edge_count,
        wall_time_per_iteration=tuple(rep.wall_time_per_iteration),
    )


def pcd_fit(x_or_gram, config, schedule=None, backend=None):
    name = default_backend_name() if backend is None else backend
    if name != "cuda-fit" or schedule is not None:
        return _orig_pcd_fit(x_or_gram, config, schedule=schedule,
                             backend="cuda" if name == "cuda-fit" else backend)
    gram = ref_solver._as_gram(x_or_gram)
    init = config.init if isinstance(config.init, str) else ours.PrecisionEstimate(config.init.omega)
    cfg = ours.SolverConfig(lam=config.lam, delta_tol=config.delta_tol,
                            max_outer_iterations=config.max_outer_iterations, init=init,
                            workers=config.workers)
    try:
        rep = ours.pcd_fit(ours.GramMatrix(gram.t, gram.n), cfg)
    except ours.NotConverged as exc:
        raise ref.NotConverged(_to_ref(exc.report)) from None
    return _to_ref(rep)


for mod in (ref_backend, ref):
    mod.available_backends = available_backends
    mod.default_backend_name = default_backend_name
    mod.get_backend = get_backend
ref_solver.get_backend = get_backend
ref_solver.pcd_fit = pcd_fit
ref.pcd_fit = pcd_fit


def pytest_report_header(config):
    return f"refsuite_plugin: B200 backends {CUDA_NAMES} registered into parconcord ({ref.__file__})"

import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))

GOLDEN = os.path.join(REPO, "tests", "golden", "reference_golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def golden():
    """Vectors recorded from the real reference package (tests/golden/make_golden.py)."""
    with np.load(GOLDEN) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def oracle():
    import oracle as o

    o.lib()
    return o


def case(golden, name):
    p, n, lam, tol = golden[f"{name}_meta"]
    return dict(p=int(p), n=int(n), lam=float(lam), tol=float(tol), t=golden[f"{name}_t"],
                x=golden[f"{name}_x"], omega=golden[f"{name}_omega"],
                iters=int(golden[f"{name}_iters"]), edges=int(golden[f"{name}_edges"]),
                delta=float(golden[f"{name}_delta"]), obj=golden[f"{name}_obj"],
                cd_omega=golden[f"{name}_cd_omega"], cd_iters=int(golden[f"{name}_cd_iters"]))

"""The C-ABI library loads and exports every symbol include/concord_pcd.h declares (no GPU needed)."""

import ctypes
import os
import re

import pytest

from paper_2106_09382_b200 import _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    text = open(os.path.join(REPO, "include", "concord_pcd.h")).read()
    return sorted(set(re.findall(r"\b(concord_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert _declared() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    for name in _declared():
        assert hasattr(L, name), name
    assert L.concord_abi_version() == _lib.ABI_VERSION


def test_no_device_is_reported_not_hidden():
    L = _lib.load()
    if _lib.device_count() > 0:
        pytest.skip("a GPU is present")
    h = ctypes.c_void_p()
    rc = L.concord_solver_create(100, 0, 0, ctypes.byref(h))
    assert rc == _lib.CONCORD_ERR_NO_DEVICE
    assert "no CUDA device" in _lib.last_error()
    import paper_2106_09382_b200 as cb

    assert cb.available_backends() == ()
    with pytest.raises(RuntimeError):
        cb.Solver(10)


@pytest.mark.parametrize("p", [256, 1000, 2000, 5000, 10000, 20000, 50000])
def test_blocked_kernel_plan_fits_every_config_size(p):
    """Host-only plan query: every BASELINE-sized problem gets the temporally blocked kernel
    (D = 4) within the 227 KB shared-memory limit -- a plan that silently falls back to the
    per-phase kernel is a large-p regression (it happened once: p >= 8000)."""
    plan = _lib.blocked_plan(p)
    assert plan["colours_per_barrier"] == 4
    assert 0 < plan["smem_bytes"] + 2048 <= 227 * 1024
    assert plan["ring_stages"] in (2, 4, 6)
    assert plan["cell_buffers"] in (1, 2)
    assert plan["ctas"] <= 148 and plan["ctas"] * plan["slab_width"] >= p
    if p <= 10000:
        assert plan["cell_buffers"] == 2  # the next block's cells are built during the colours


def test_blocked_plan_small_p_uses_per_phase_kernel():
    assert _lib.blocked_plan(100)["colours_per_barrier"] == 0

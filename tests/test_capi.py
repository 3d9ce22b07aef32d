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

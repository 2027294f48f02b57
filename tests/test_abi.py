"""The C-ABI library loads without a GPU and exports every entry point
declared in include/sdmrg_b200.h (no compute calls here)."""

import os
import re

from conftest import ROOT


def declared_functions():
    src = open(os.path.join(ROOT, "include", "sdmrg_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sdmrg_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_bound_functions():
    from paper_2305_05581_b200 import _lib
    assert declared_functions() == sorted(_lib.EXPORTED)


def test_library_exports_every_declared_symbol():
    from paper_2305_05581_b200 import _lib
    lib = _lib.load(rebuild=False)
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.sdmrg_version() >= 1
    assert lib.sdmrg_launch_count() >= 0


def test_argument_errors_mirror_reference_exceptions():
    """Bad arguments fail loudly without touching a device (ValueError /
    WorkspaceError mapping of sbmm4s.py:25)."""
    import ctypes

    import pytest

    from paper_2305_05581_b200 import _lib
    lib = _lib.load(rebuild=False)
    with pytest.raises(_lib.SdmrgError):
        _lib.check(lib.sdmrg_dgemm(0, 0, -1, 2, 2, 1.0, None, 1, None, 1, 0.0, None, 1, None))
    with pytest.raises(_lib.WorkspaceError):
        _lib.check(lib.sdmrg_sbmm4s(4, 4, 4, 4, 2, 1.0, None, 4, None, 4, 16, None, 4, 16,
                                    None, 4, None, 3, None, None))
    with pytest.raises(_lib.SdmrgError):
        _lib.check(lib.sdmrg_plan_build(None, ctypes.byref(ctypes.c_void_p())))

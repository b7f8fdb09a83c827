"""The C-ABI library loads and exports every symbol include/ridc_b200.h declares
(no compute calls: runs without a GPU)."""

import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "ridc_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ridc_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("ridc_create", "ridc_run", "ridc_run_device", "ridc_destroy", "ridc_last_error",
              "ridc_op_apply", "ridc_op_solve", "ridc_op_step", "ridc_pipe_create",
              "ridc_pipe_run_interval"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_1209_4297_b200 import _lib
    L = _lib.lib()
    for s in declared_symbols():
        assert hasattr(L, s), s
        assert s in _lib.SIGNATURES, f"{s} missing from the ctypes table"


def test_struct_layout_matches_header():
    from paper_1209_4297_b200.problems import CProblem
    assert ctypes.sizeof(CProblem) == 4 * 4 + 7 * 8
    from paper_1209_4297_b200._lib import RidcInfo
    assert ctypes.sizeof(RidcInfo) == 4 + 4 + 8 + 8 + 8 + 4 * 4 + 8 + 8 + 8 + 4 + 4   # ..., path, fell_back


def test_create_rejects_bad_config_without_gpu():
    """Validation happens before any CUDA call (RidcConfig semantics)."""
    from paper_1209_4297_b200 import _lib, problems as P
    from paper_1209_4297_b200.errors import ConfigError, DimensionMismatch
    import pytest
    L = _lib.lib()
    pd = P.adv_diff_desk().problem.to_c()
    h = ctypes.c_void_p()
    rc = L.ridc_create(ctypes.byref(pd), 0.0, 1.0, 4, 10, 1, None, 0, 0, 0, ctypes.byref(h))
    with pytest.raises(ConfigError):
        _lib.check(rc)
    bad = P.adv_diff_desk().problem.to_c()
    bad.ny = 2
    rc = L.ridc_create(ctypes.byref(bad), 0.0, 1.0, 1, 10, 1, None, 0, 0, 0, ctypes.byref(h))
    with pytest.raises(DimensionMismatch):
        _lib.check(rc)

"""The C-ABI library loads without a GPU and exports every entry point that
include/ss_abi.h declares (no compute calls here)."""

import ctypes
import os
import re

from paper_2605_05876_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "ss_abi.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ss_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "ss_preprocess" in syms and "ss_raster_backward" in syms and len(syms) >= 18


def test_library_exports_every_declared_symbol():
    lib = _lib.load(require_cuda=False)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_covers_header():
    assert set(declared_symbols()) <= set(_lib.EXPORTED)


def test_version_and_error_string():
    lib = _lib.load(require_cuda=False)
    assert lib.ss_version() >= 1
    assert isinstance(lib.ss_last_error(), bytes)


def test_invalid_arguments_rejected_before_launch():
    """Host-side argument validation returns SS_ERR_INVALID without a GPU."""
    lib = _lib.load(require_cuda=False)
    assert lib.ss_adam_step(10, None, None, None, None, 0, 0.1, 0.9, 0.999, 1e-15, None) == _lib.SS_ERR_INVALID
    assert lib.ss_brdf_lut(1, 8, None, None) == _lib.SS_ERR_INVALID
    bg, _keep = _lib.fvec([0, 0, 0])
    assert lib.ss_raster_forward(0, 10, 16, None, None, None, None, bg, 16, None, None, None, None, None, None,
                                 None, None) == _lib.SS_ERR_INVALID

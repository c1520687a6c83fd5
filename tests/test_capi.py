"""The C-ABI library builds for sm_100a, loads without a GPU and exports every
symbol include/contour.h declares.  CPU only (no compute calls)."""

import os
import re
import subprocess

import pytest

from paper_2311_02811_b200 import _lib, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _lib.load()


def header_symbols():
    text = open(os.path.join(ROOT, "include", "contour.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cc_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_expected_entry_points():
    syms = header_symbols()
    for s in ("cc_create", "cc_destroy", "cc_stage_edges", "cc_run", "cc_sweep", "cc_compress",
              "cc_early_check", "cc_last_error", "cc_gen_rmat_device"):
        assert s in syms


def test_every_header_symbol_exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (cc_[a-z0-9_]+)", out))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing
    for s in header_symbols():
        assert hasattr(lib, s)
        assert s in _lib.SIGNATURES, f"{s} lacks a ctypes signature"


def test_built_for_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_version_and_error_path_without_gpu(lib):
    assert lib.cc_version() == 1
    import ctypes
    h = ctypes.c_void_p()
    rc = lib.cc_create(0, None, ctypes.byref(h))
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        assert rc != 0 and not h.value
        assert _lib.last_error()
    else:
        assert rc == 0
        lib.cc_destroy(h)


def test_error_mapping():
    from paper_2311_02811_b200.errors import IterationCapExceeded
    with pytest.raises(ValueError):
        _lib.check(_lib.CC_EINVAL, "x")
    with pytest.raises(IterationCapExceeded):
        _lib.check(_lib.CC_ECAP, "x")
    with pytest.raises(RuntimeError):
        _lib.check(_lib.CC_ECUDA, "x")

"""The C-ABI library loads and exports every symbol include/sellb.h declares
(no compute calls: runs on CPU-only hosts)."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "sellb.h")
LIB = os.path.join(REPO, "paper_1307_6209_b200", "libsellb200.so")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sellb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("sellb_build_from_crs", "sellb_spmv", "sellb_spmv_host",
                 "sellb_spmv_sell_range_host", "sellb_export", "sellb_free",
                 "sellb_last_error"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "build first: make -C paper_1307_6209_b200/csrc"
    lib = ctypes.CDLL(LIB)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_covers_header():
    from paper_1307_6209_b200 import _lib
    assert sorted(_lib.EXPORTED) == declared_symbols()
    _lib.load()


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_error_string_and_param_error_without_device():
    """Parameter checks run before any device work and report through the
    thread-local error string."""
    from paper_1307_6209_b200 import _lib
    lib = _lib.load()
    out = ctypes.c_void_p()
    rc = lib.sellb_build_from_crs(None, None, None, 0, 4, 4, 0, 1, 1, 0, 0, None, 0,
                                  ctypes.byref(out))
    assert rc == -1
    assert "chunk height" in _lib.last_error()
    rc = lib.sellb_build_from_crs(None, None, None, 0, 4, 4, 4, 1, 32, 0, 0, None, 0,
                                  ctypes.byref(out))
    assert rc == -1 and "align_bytes" in _lib.last_error()


def test_product_path_fails_loudly_without_gpu():
    from paper_1307_6209_b200 import _lib, ResourceError
    if _lib.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(ResourceError):
        _lib.require_device()

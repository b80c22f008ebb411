"""The C-ABI library loads and exports every symbol include/gridlq_b200.h declares
(no compute calls: CPU tier)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT


def _declared():
    hdr = open(os.path.join(ROOT, "include", "gridlq_b200.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(gq_[a-z_]+)\s*\(", hdr)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2304_04980_b200 import _lib
    from paper_2304_04980_b200.build import build

    if not os.path.exists(_lib.LIB_PATH):
        build()
    return _lib.LIB_PATH


def test_exports_match_header(lib_path):
    lib = ctypes.CDLL(lib_path)
    names = _declared()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    from paper_2304_04980_b200 import _lib

    assert set(_lib.EXPORTS) == set(names)


def test_binding_loads_without_gpu(lib_path):
    from paper_2304_04980_b200 import _lib

    lib = _lib.load()
    assert b"sm_100a" in lib.gq_version()
    # a null descriptor is rejected with INVALID_ARG before any CUDA call
    assert lib.gq_create(None, 2, 2, None) == _lib.GQ_INVALID_ARG
    assert "null" in _lib.last_error()


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    from paper_2304_04980_b200 import _lib

    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.load()

"""The C-ABI library loads and exports every function declared in include/bddcso_b200.h
(no GPU needed: nothing is called)."""
import ctypes
import os
import re

import pytest

from conftest import ROOT


def _declared():
    hdr = open(os.path.join(ROOT, "include", "bddcso_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|long long|double|const double\s*\*)\s*(bddc_\w+)\s*\(", hdr, re.M)))


def test_header_lists_entry_points():
    names = _declared()
    for n in ("bddc_create", "bddc_setup", "bddc_apply", "bddc_pcg", "bddc_spmv", "bddc_destroy"):
        assert n in names


def test_library_exports_all_symbols():
    from paper_2001_07289_b200 import _capi

    if not os.path.exists(_capi.LIB_PATH):
        pytest.skip("library not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(_capi.LIB_PATH)
    for n in _declared():
        assert hasattr(lib, n), n
    assert set(_capi.EXPORTS) == set(_declared())


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    from paper_2001_07289_b200 import _capi

    monkeypatch.setattr(_capi, "_lib", None)
    monkeypatch.setattr(_capi, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _capi.load()

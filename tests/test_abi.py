"""The C-ABI library loads on a CPU host and exports exactly what include/prefillonly.h declares."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_2505_07203_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "prefillonly.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(po_\w+)\(", text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.SIGNATURES), "ctypes signatures out of sync with the header"


def test_version_and_error_text():
    lib = _lib.load()
    assert b"sm_100a" in lib.po_version()
    # argument validation runs on the host, without touching a GPU
    rc = lib.po_op_gemm(None, 0, None, 0, None, 0, None, 0, 1, 256, 64, 0, None, 0, 0, None)
    assert rc == _lib.PO_ERR_ARG
    assert b"null" in lib.po_last_error()
    rc = lib.po_engine_info(None, None, 0)
    assert rc == _lib.PO_ERR_ARG


def test_sm100a_cubin_embedded():
    data = _lib.lib_path().read_bytes()
    assert b"sm_100a" in data or b"sm_100" in data


def test_no_cpu_fallback_when_library_missing(monkeypatch, tmp_path):
    monkeypatch.setenv("PREFILLONLY_LIB", str(tmp_path / "missing.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(_lib.PrefillOnlyError):
        _lib.load()

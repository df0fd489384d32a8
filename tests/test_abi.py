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


def test_host_validation_of_configs_and_ops():
    """Configuration and argument errors are reported before any CUDA call, with the reference's error taxonomy."""
    from dataclasses import replace

    from paper_2505_07203_b200.config import LLAMA_3_1_8B, TINY, to_c_cfg

    lib = _lib.load()
    eng = ctypes.c_void_p()
    for bad, needle in ((replace(TINY, head_dim=64), b"head_dim"), (replace(TINY, n_kv_heads=3), b"multiple"),
                        (replace(TINY, hidden=250), b"256"), (replace(LLAMA_3_1_8B, hidden=16384), b"8192"),
                        (replace(TINY, num_layers=0), b"positive")):
        cfg = to_c_cfg(bad, max_tokens=1024)
        assert lib.po_init(0, ctypes.addressof(cfg), 0, ctypes.addressof(eng)) == _lib.PO_ERR_CONFIG
        assert needle in lib.po_last_error(), lib.po_last_error()
        assert not eng.value
    # op entry points: shapes and pointers checked on the host
    assert lib.po_op_gemm_fp8(None, 0, None, None, 0, None, None, 0, None, 0, 128, 256, 128, 0, None, 0, 0,
                              None) == _lib.PO_ERR_ARG
    x = ctypes.c_void_p(16)  # never dereferenced: validation fails first
    assert lib.po_op_gemm_fp8(x, 128, x, x, 128, x, x, 256, None, 0, 128, 256, 64, 0, None, 0, 0, None) == _lib.PO_ERR_ARG
    assert b"K%128" in lib.po_last_error()
    assert lib.po_op_quantize_e4m3(x, 8, 4, 24, x, 32, x, None) == _lib.PO_ERR_ARG  # cols % 16
    assert lib.po_op_attention(x, 6144, 100, 100, 32, 8, x, 4096, None) == _lib.PO_ERR_ARG  # q_offset == n_total
    assert lib.po_op_attention(x, 6144, 100, 0, 30, 8, x, 4096, None) == _lib.PO_ERR_ARG  # 30 % 8
    assert lib.po_prefill(None, None, 0, 0, None, 0, None, 0, None, None, None, None) == _lib.PO_ERR_ARG

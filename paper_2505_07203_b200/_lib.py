"""ctypes binding of libprefillonly.so (the C-ABI declared in include/prefillonly.h).

The shared library is built in-tree by `make` (see __graft_entry__.build). There is no CPU or
PyTorch fallback: if the library is missing, every call fails loudly.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_LIB_PATH = Path(__file__).with_name("libprefillonly.so")
_lib = None


class PrefillOnlyError(RuntimeError):
    """Raised when a C-ABI call returns a non-zero status."""

    def __init__(self, code: int, message: str):
        super().__init__(f"[{code}] {message}")
        self.code = code


# status codes (include/prefillonly.h)
PO_ERR_CONFIG = -2
PO_ERR_CAPACITY = -3
PO_ERR_CUDA = -4
PO_ERR_ARG = -5
PO_ERR_POOL = -6

# GEMM epilogues
EPI_BF16 = 0
EPI_RESID_F32 = 1
EPI_SILU_MUL = 2
EPI_QKV_ROPE = 3
EPI_F32 = 4

_VP = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64

# name -> (restype, argtypes); every symbol here must be exported by the .so
SIGNATURES = {
    "po_last_error": (ctypes.c_char_p, []),
    "po_version": (ctypes.c_char_p, []),
    "po_init": (_I32, [_I32, _VP, ctypes.c_uint64, _VP]),
    "po_free": (_I32, [_VP]),
    "po_prefill": (_I32, [_VP, _VP, _I32, _I32, _VP, _I32, _VP, _I32, _VP, _VP, _VP, _VP]),
    "po_last_service_ms": (_I32, [_VP, _VP]),
    "po_prefill_submit": (_I32, [_VP, _VP, _I32, _I32, _VP, _I32, _VP, _I32, _VP, _VP]),
    "po_prefill_query": (_I32, [_VP, _I64, _VP]),
    "po_prefill_wait": (_I32, [_VP, _I64, _VP, _VP, _VP, _VP]),
    "po_prefill_device": (_I32, [_VP, _VP, _I32, _I32, _VP, _I32, _VP, _I32, _VP, _VP, _VP, _VP]),
    "po_engine_stream": (_I32, [_VP, _VP]),
    "po_last_launches": (_I32, [_VP, _VP]),
    "po_profile_begin": (_I32, [_VP]),
    "po_profile_end": (_I32, [_VP, _VP, _VP, _I32]),
    "po_pool_evict": (_I32, [_VP, _VP, _I32]),
    "po_engine_info": (_I32, [_VP, _VP, _I32]),
    "po_load_weight": (_I32, [_VP, _I32, _I32, _VP, _I64]),
    "po_op_attention": (_I32, [_VP, _I64, _I32, _I32, _I32, _I32, _VP, _I64, _VP]),
    "po_op_gemm": (_I32, [_VP, _I64, _VP, _I64, _VP, _I64, _VP, _I64, _I32, _I32, _I32, _I32, _VP, _I32, _I32, _VP]),
    "po_op_gemm_fp8": (_I32, [_VP, _I64, _VP, _VP, _I64, _VP, _VP, _I64, _VP, _I64, _I32, _I32, _I32, _I32, _VP, _I32,
                              _I32, _VP]),
    "po_op_quantize_e4m3": (_I32, [_VP, _I64, _I32, _I32, _VP, _I64, _VP, _VP]),
    "po_op_stream_gemm": (_I32, [_VP, _I64, _VP, _I64, _VP, _I64, _I32, _I32, _I32, _VP, _I64, _VP, _I64, _I32, _VP]),
}


def lib_path() -> Path:
    return Path(os.environ.get("PREFILLONLY_LIB", _LIB_PATH))


def load():
    """Load the shared library once; raise if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    path = lib_path()
    if not path.is_file():
        raise PrefillOnlyError(PO_ERR_CUDA, f"{path} not built; run `make` (or __graft_entry__.build())")
    lib = ctypes.CDLL(str(path))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int):
    if rc != 0:
        msg = load().po_last_error().decode(errors="replace")
        raise PrefillOnlyError(rc, msg)


def call(name: str, *args):
    check(getattr(load(), name)(*args))

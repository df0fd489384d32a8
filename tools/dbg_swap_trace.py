"""Per-CTA timeline of one swap-AB GEMM launch (needs a -DSWAP_TRACE build:
tools/build_variant.sh swaptrace gemm_swap.cu -DSWAP_TRACE; PREFILLONLY_LIB=build/variants/lib_swaptrace.so).
python tools/dbg_swap_trace.py M N K [flush]"""
import ctypes
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2505_07203_b200 import _lib  # noqa: E402

lib = _lib.load()
M, N, K = [int(x) for x in sys.argv[1:4]]
flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda")
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
B = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
for _ in range(3):
    flush.sum()
    torch.cuda.synchronize()
    _lib.call("po_op_gemm", p(A), K, p(B), K, p(out), N, None, 0, M, N, K, 0, None, 0, 0, None)
    torch.cuda.synchronize()
buf = (ctypes.c_uint64 * (296 * 16))()
lib.po_debug_swap_trace(ctypes.addressof(buf))
arr = [list(buf[i * 16:(i + 1) * 16]) for i in range(296)]
arr = [a for a in arr if a[0]]
names = ["start", "setup_done", "first_full", "last_commit", "epi_start", "epi_done", "exit", "last_epi"] + [f"c{c}_{w}" for c in range(2) for w in ("ld", "buf", "staged", "fenced")]
t0 = min(a[0] for a in arr)
print(f"M={M} N={N} K={K}: {len(arr)} CTAs; us after the first CTA start (min / median / max)")
for i, nm in enumerate(names):
    v = [(a[i] - t0) / 1e3 for a in arr if a[i]]
    if v:
        print(f"  {nm:12s} {min(v):7.2f} {statistics.median(v):7.2f} {max(v):7.2f}")

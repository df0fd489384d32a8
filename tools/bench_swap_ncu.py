"""One launch of each Llama-3.1-8B prefix-hit GEMM shape (M = 160) through po_op_gemm, for an ncu launch list
(gemm kernel and split-K reduce separately): python tools/bench_swap_ncu.py"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2505_07203_b200 import _lib  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 160
SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336)}
flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda")
p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
for name, (N, K) in SHAPES.items():
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    for _ in range(3):
        flush.sum()
        _lib.call("po_op_gemm", p(A), K, p(B), K, p(out), N, None, 0, M, N, K, 0, None, 0, 0, None)
    torch.cuda.synchronize()

"""Weight-streaming kernel vs the per-GEMM split-K launches on the Llama-3.1-8B prefix-hit shapes (M = 160).

python tools/bench_stream.py   -> per shape: stream us, per-GEMM us, weight GB/s of each (CUDA events, 50 reps,
an L2-flushing read between reps so the weights come from HBM as in a forward).
"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2505_07203_b200 import _lib  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 160
SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336)}
flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda")


def p(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def timed(fn, reps=50):
    ts = []
    for _ in range(reps):
        flush.sum()  # read-based L2 flush (a write flush leaves dirty lines)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


for name, (N, K) in SHAPES.items():
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    st = lambda: _lib.call("po_op_stream_gemm", p(A), K, p(B), K, p(out), N, M, N, K, None, 0, None, 0, 0, None)  # noqa
    pg = lambda: _lib.call("po_op_gemm", p(A), K, p(B), K, p(out), N, None, 0, M, N, K, 0, None, 0, 0, None)  # noqa
    t_s, t_g = timed(st), timed(pg)
    wb = N * K * 2
    print(f"{name:8s} M={M} N={N} K={K}: stream {t_s:7.1f} us ({wb / t_s / 1e3:6.0f} GB/s)   "
          f"per-GEMM {t_g:7.1f} us ({wb / t_g / 1e3:6.0f} GB/s)", flush=True)

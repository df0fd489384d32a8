"""Per-CTA timeline of the last stream-K GEMM launch of shape N (M > 1) inside warm prefix-hit forwards (needs a
tools/build_variant.sh skt<N> gemm_sk.cu "-DSK_TRACE -DSK_TRACE_N=<N>" build):
PREFILLONLY_LIB=build/variants/lib_skt<N>.so python tools/dbg_sk_trace.py"""
import ctypes
import statistics
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2505_07203_b200 import _lib  # noqa: E402
from paper_2505_07203_b200.config import LLAMA_3_1_8B as M  # noqa: E402
from paper_2505_07203_b200.engine import Engine  # noqa: E402

n = 20000
e = Engine(M, seed=0, max_tokens=20480, pool_blocks=1400)
toks = np.random.default_rng([0, 0, 0]).integers(0, 2 ** 32, size=n, dtype=np.uint32)
slots = list(range(n // 16))
e.prefill(toks, [9642, 2822], 0, slots)
for _ in range(4):
    e.prefill(toks, [9642, 2822], (n - 160) // 16 * 16, slots)
buf = (ctypes.c_uint64 * (296 * 16))()
buf0 = list(buf)
_lib.load().po_debug_swap_trace(ctypes.addressof(buf))
arr = [list(buf[i * 16:(i + 1) * 16]) for i in range(296)]
arr = [a for a in arr if a[0]]
names = ["start", "setup", "first_full", "last_commit", "epi_first", "tail_pub", "flags_seen", "fix_start",
         "epi_done", "exit", "fx0_land", "fx0_r8", "fx0_done", "fx1_land", "fx1_r8", "fx1_done"]
t0 = min(a[0] for a in arr)
print(f"{len(arr)} CTAs; us after the first CTA start (min / median / max, count)")
for i, nm in enumerate(names):
    v = [(a[i] - t0) / 1e3 for a in arr if a[i] >= t0 and a[i] - t0 < 10**6]
    if v:
        print(f"  {nm:12s} {min(v):7.2f} {statistics.median(v):7.2f} {max(v):7.2f}  {len(v)}")
if len(sys.argv) > 1:
    for k, a in enumerate(arr):
        print(k, " ".join(f"{(x - t0) / 1e3:6.1f}" if x >= t0 else "   -  " for x in a[:16]))

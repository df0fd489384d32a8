"""Per-CTA timeline of the last swap-AB launch of shape N (M > 1) inside warm prefix-hit forwards (needs a
-DSWAP_TRACE -DSWAP_TRACE_N=<N> build): PREFILLONLY_LIB=... python tools/dbg_swap_trace_hit.py"""
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
_lib.load().po_debug_swap_trace(ctypes.addressof(buf))
arr = [list(buf[i * 16:(i + 1) * 16]) for i in range(296)]
arr = [a for a in arr if a[0]]
names = ["start", "setup_done", "first_full", "last_commit", "epi_start", "epi_done", "exit", "last_epi"] + [f"c{c}_{w}" for c in range(2) for w in ("ld", "buf", "staged", "fenced")]
t0 = min(a[0] for a in arr)
print(f"{len(arr)} CTAs; us after the first CTA start (min / median / max)")
for i, nm in enumerate(names):
    v = [(a[i] - t0) / 1e3 for a in arr if a[i] >= t0]
    if v:
        print(f"  {nm:12s} {min(v):7.2f} {statistics.median(v):7.2f} {max(v):7.2f}")

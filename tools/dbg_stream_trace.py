"""Debug: grid-barrier trace of one two-phase po_op_stream_gemm launch (needs a -DSTREAM_DBG_TRACE build)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2505_07203_b200 import _lib  # noqa: E402

lib = _lib.load()
M, N1, K, N2 = [int(x) for x in sys.argv[1:5]] if len(sys.argv) > 4 else (200, 1024, 1024, 512)
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
B1 = (torch.randn(N1, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
B2 = (torch.randn(max(N2, 256), N1, device="cuda") / N1 ** 0.5).to(torch.bfloat16)
o1 = torch.full((M, N1), float("nan"), dtype=torch.bfloat16, device="cuda")
o2 = torch.empty(M, max(N2, 256), dtype=torch.bfloat16, device="cuda")
p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa
_lib.call("po_op_stream_gemm", p(A), K, p(B1), K, p(o1), N1, M, N1, K, p(B2) if N2 else None, N1, p(o2), max(N2, 256),
          N2, None)
torch.cuda.synchronize()
buf = (ctypes.c_uint64 * (148 * 16))()
lib.po_debug_stream_trace(ctypes.addressof(buf))
arr = [list(buf[i * 16:(i + 1) * 16]) for i in range(148)]
names = ["start", "prod_done", "first_tfull", "last_tfull", "dumps_done", "flags_ok", "reduce_done", "arrive",
         "b0_land", "b1_land", "b2_land", "b3_land", "b4_land", "t0_end", "t1_flags", "t1_end", "b1_issue"]
t0 = min(a[0] for a in arr if a[0])
import statistics
for i, nm in enumerate(names):
    v = [(a[i] - t0) / 1e3 for a in arr if a[i]]
    if v:
        print(f"{nm:12s} n={len(v):3d} min {min(v):7.2f} med {statistics.median(v):7.2f} max {max(v):7.2f} us")
print("o2 nan", torch.isnan(o2.float()).sum().item(), "o1 nan", torch.isnan(o1.float()).sum().item())
ref = o1.float() @ B2.float().T if N2 else o2.float()
print("o2 max err", (o2.float() - ref).abs().max().item())

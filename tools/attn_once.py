"""One po_op_attention launch (after two warm-ups) at Llama-3.1-8B head shapes, for ncu captures:
python tools/attn_once.py n [q_offset]"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2505_07203_b200 import _lib  # noqa: E402

n = int(sys.argv[1])
off = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hq, hkv = 32, 8
ld = (hq + 2 * hkv) * 128
qkv = torch.randn(n, ld, device="cuda").to(torch.bfloat16)
out = torch.empty(n - off, hq * 128, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    _lib.call("po_op_attention", ctypes.c_void_p(qkv.data_ptr()), ld, n, off, hq, hkv, ctypes.c_void_p(out.data_ptr()),
              hq * 128, None)
torch.cuda.synchronize()
print("ok", n, off)

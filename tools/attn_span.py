"""Per-CTA spans (globaltimer at entry / after setup / exit, with the CTA's KV split and query unit) of one
attention launch from a -DATTN_SPAN build, L2 flushed first:
  tools/build_variant.sh span attention.cu "-DATTN_SPAN"
  PREFILLONLY_LIB=build/variants/lib_span.so python tools/attn_span.py [n] [n_miss]"""
import collections
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2505_07203_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
n_miss = int(sys.argv[2]) if len(sys.argv) > 2 else 160
hq, hkv = 32, 8
ld = (hq + 2 * hkv) * 128
qkv = torch.randn(n, ld, device="cuda").to(torch.bfloat16)
out = torch.empty(n_miss, hq * 128, dtype=torch.bfloat16, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
lib = _lib.load()
for _ in range(3):
    flush.sum()
    _lib.call("po_op_attention", ctypes.c_void_p(qkv.data_ptr()), ld, n, n - n_miss, hq, hkv,
              ctypes.c_void_p(out.data_ptr()), hq * 128, None)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (8192 * 4))()
assert lib.po_debug_attn_span(buf, 8192 * 4) == 0
t = np.frombuffer(buf, dtype=np.uint64).reshape(8192, 4)
live = np.nonzero(t[:, 2])[0]
t0 = t[live, 0].min()
st = (t[live, 0] - t0) / 1e3
su = (t[live, 1] - t0) / 1e3
en = (t[live, 2] - t0) / 1e3
split = (t[live, 3] >> 32).astype(int)
unit = (t[live, 3] & 0xffffffff).astype(int)
print(f"{len(live)} CTAs, kernel span {en.max():.2f} us; start max {st.max():.2f}, setup median {np.median(su - st):.2f}")
print(f"duration (exit - start) min / median / max: {np.min(en - st):.2f} / {np.median(en - st):.2f} / "
      f"{np.max(en - st):.2f} us")
g = collections.defaultdict(list)
for i in range(len(live)):
    g[("split", split[i])].append(en[i] - st[i])
    g[("unit", unit[i])].append(en[i] - st[i])
for k in sorted(g):
    v = np.array(g[k])
    print(f"  {k[0]} {k[1]:3d}: {len(v):4d} CTAs  duration median {np.median(v):7.2f}  max {v.max():7.2f} us")
order = np.argsort(en)[-8:]
print("last CTAs to exit (block, split, unit, start, exit):",
      [(int(live[i]), int(split[i]), int(unit[i]), round(float(st[i]), 2), round(float(en[i]), 2)) for i in order])

"""Per-tile timeline of one attention CTA of a prefix-hit launch (short packed query, split-KV) from a -DATTN_TRACE=b
build: kernel entry, setup done, each tile's S-ready / P-done per slot, partial-output stores done (SM cycles).

  tools/build_variant.sh trace0 attention.cu "-DATTN_TRACE=0"
  PREFILLONLY_LIB=build/variants/lib_trace0.so python tools/attn_trace_hit.py [n] [n_miss]
"""
import ctypes
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2505_07203_b200 import _lib  # noqa: E402

EV, TILES = 24, 512


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
    n_miss = int(sys.argv[2]) if len(sys.argv) > 2 else 160
    hq, hkv = 32, 8
    ld = (hq + 2 * hkv) * 128
    q0 = n - n_miss
    qkv = torch.randn(n, ld, device="cuda").to(torch.bfloat16)
    out = torch.empty(n_miss, hq * 128, dtype=torch.bfloat16, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    lib = _lib.load()
    for _ in range(3):
        flush.sum()  # K/V cold in L2, as in a hit forward (the prefix was written long ago)
        _lib.call("po_op_attention", ctypes.c_void_p(qkv.data_ptr()), ld, n, q0, hq, hkv,
                  ctypes.c_void_p(out.data_ptr()), hq * 128, None)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (EV * TILES))()
    assert lib.po_debug_attn_trace(buf, EV * TILES) == 0
    t = np.frombuffer(buf, dtype=np.uint64).reshape(EV, TILES).astype(np.int64)
    t0 = t[21, 0]
    nt = int(np.count_nonzero(t[1]))
    rel = lambda x: int(x - t0) if x else None  # noqa: E731
    rep = {"setup_done": rel(t[21, 1]), "tiles": nt,
           "slot0_S_ready": [rel(t[1, j]) for j in range(nt)],
           "slot1_S_ready": [rel(t[5, j]) for j in range(nt)],
           "slot0_P_done": [rel(t[3, j]) for j in range(nt)],
           "stores_done": [rel(t[22, 0]), rel(t[23, 0])]}
    d = np.diff(t[1, :nt])
    rep["period_median"] = float(np.median(d)) if len(d) else None
    print(json.dumps(rep))


if __name__ == "__main__":
    main()

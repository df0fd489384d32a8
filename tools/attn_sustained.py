"""Sustained attention throughput (CUDA events over many back-to-back launches, so the clocks settle under the power
cap) of po_op_attention and cuDNN SDPA, alternating: python tools/attn_sustained.py n iters rounds"""
import ctypes
import json
import subprocess
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, ".")
from paper_2505_07203_b200 import _lib  # noqa: E402

n, iters, rounds = (int(x) for x in sys.argv[1:4])
hq, hkv = 32, 8
ld = (hq + 2 * hkv) * 128
qkv = torch.randn(n, ld, device="cuda").to(torch.bfloat16)
out = torch.empty(n, hq * 128, dtype=torch.bfloat16, device="cuda")
q = qkv[:, :hq * 128].view(n, hq, 128).transpose(0, 1)[None]
k = qkv[:, hq * 128:(hq + hkv) * 128].view(n, hkv, 128).transpose(0, 1)[None]
v = qkv[:, (hq + hkv) * 128:].view(n, hkv, 128).transpose(0, 1)[None]
ours = lambda: _lib.call("po_op_attention", ctypes.c_void_p(qkv.data_ptr()), ld, n, 0, hq, hkv,
                         ctypes.c_void_p(out.data_ptr()), hq * 128, None)
cudnn = lambda: F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
fl = 4.0 * 128 * hq * n * n / 2


def clk():
    try:
        return int(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits", "-i", "0"],
                                  capture_output=True, text=True).stdout.split()[0])
    except Exception:
        return -1


with torch.nn.attention.sdpa_kernel(torch.nn.attention.SDPBackend.CUDNN_ATTENTION):
    for f in (ours, cudnn):
        f()
    torch.cuda.synchronize()
    for r in range(rounds):
        for name, f in (("ours", ours), ("cudnn", cudnn)):
            s, e = torch.cuda.Event(True), torch.cuda.Event(True)
            s.record()
            for _ in range(iters):
                f()
            e.record()
            c = clk()
            torch.cuda.synchronize()
            t = s.elapsed_time(e) / iters
            print(json.dumps({"n": n, "impl": name, "round": r, "ms": round(t, 3), "tflops": round(fl / t / 1e9, 1),
                              "sm_mhz_late": c}), flush=True)

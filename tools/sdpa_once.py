"""One cuDNN SDPA launch (after warm-ups) at Llama-3.1-8B head shapes, for ncu captures: python tools/sdpa_once.py n"""
import sys

import torch
import torch.nn.functional as F

n = int(sys.argv[1])
hq, hkv = 32, 8
qkv = torch.randn(n, (hq + 2 * hkv) * 128, device="cuda").to(torch.bfloat16)
q = qkv[:, :hq * 128].view(n, hq, 128).transpose(0, 1)[None]
k = qkv[:, hq * 128:(hq + hkv) * 128].view(n, hkv, 128).transpose(0, 1)[None]
v = qkv[:, (hq + hkv) * 128:].view(n, hkv, 128).transpose(0, 1)[None]
with torch.nn.attention.sdpa_kernel(torch.nn.attention.SDPBackend.CUDNN_ATTENTION):
    for _ in range(3):
        F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
torch.cuda.synchronize()
print("ok", n)

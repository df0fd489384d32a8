"""CUDA-event timing of po_op_attention at Llama-3.1-8B head shapes (32 q / 8 kv heads, d=128)."""
import ctypes, sys, json
import torch
sys.path.insert(0, ".")
from paper_2505_07203_b200 import _lib

def p(t): return ctypes.c_void_p(t.data_ptr())

def run(n, off=0, hq=32, hkv=8, iters=5):
    ld = (hq + 2 * hkv) * 128
    qkv = torch.randn(n, ld, device="cuda").to(torch.bfloat16)
    out = torch.empty(n - off, hq * 128, dtype=torch.bfloat16, device="cuda")
    f = lambda: _lib.call("po_op_attention", p(qkv), ld, n, off, hq, hkv, p(out), hq * 128, None)
    for _ in range(2): f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(iters): f()
    e.record(); torch.cuda.synchronize()
    t = s.elapsed_time(e) / iters
    fl = 4.0 * 128 * hq * (n * n - off * off) / 2
    q = qkv[:, :hq*128].view(n, hq, 128).transpose(0, 1)[None]
    k = qkv[:, hq*128:(hq+hkv)*128].view(n, hkv, 128).transpose(0, 1)[None]
    v = qkv[:, (hq+hkv)*128:].view(n, hkv, 128).transpose(0, 1)[None]
    import torch.nn.functional as F
    try:
        for _ in range(2): F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
        s.record()
        for _ in range(iters): F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
        e.record(); torch.cuda.synchronize()
        tr = s.elapsed_time(e) / iters
    except Exception as ex:
        tr = float("nan")
    print(json.dumps({"n": n, "off": off, "ms": round(t, 3), "tflops": round(fl / t / 1e9, 1),
                      "sdpa_ms": round(tr, 3), "sdpa_tflops": round(fl / tr / 1e9, 1)}), flush=True)

if __name__ == "__main__":
    run(4096); run(20000); run(20000, 19840); run(65536, iters=2)

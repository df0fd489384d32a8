"""Causal GQA prefill attention at Llama-3.1-8B head shapes (32 q / 8 kv heads, d=128, bf16): this repo's tcgen05
kernel (po_op_attention) next to the library kernels available in the image, on the same inputs, CUDA events,
median of `iters` launches after warm-up. One JSON line per (n, implementation). Libraries are evidence only; none
is on the product path.

  python tools/attn_vs_libs.py [n ...]      (default 4096 20000 65536)
"""
import ctypes
import json
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, ".")
from paper_2505_07203_b200 import _lib  # noqa: E402

HQ, HKV, D = 32, 8, 128


def p(t):
    return ctypes.c_void_p(t.data_ptr())


def timed(fn, iters):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


def main(sizes):
    dev = torch.cuda.get_device_name()
    for n in sizes:
        iters = 10 if n <= 20000 else 3
        ld = (HQ + 2 * HKV) * D
        qkv = (torch.randn(n, ld, device="cuda") * 0.5).to(torch.bfloat16)
        out = torch.empty(n, HQ * D, dtype=torch.bfloat16, device="cuda")
        flops = 4.0 * D * HQ * n * n / 2
        q = qkv[:, :HQ * D].view(n, HQ, D)
        k = qkv[:, HQ * D:(HQ + HKV) * D].view(n, HKV, D)
        v = qkv[:, (HQ + HKV) * D:].view(n, HKV, D)
        impls = {"prefillonly_tcgen05": lambda: _lib.call("po_op_attention", p(qkv), ld, n, 0, HQ, HKV, p(out),
                                                          HQ * D, None)}
        qt, kt, vt = (x.transpose(0, 1).contiguous()[None] for x in (q, k, v))
        ke, ve = kt.repeat_interleave(HQ // HKV, dim=1), vt.repeat_interleave(HQ // HKV, dim=1)
        from torch.nn.attention import SDPBackend, sdpa_kernel

        for name, be in (("torch_sdpa_cudnn", SDPBackend.CUDNN_ATTENTION),
                         ("torch_sdpa_flash", SDPBackend.FLASH_ATTENTION)):
            def f(be=be):
                with sdpa_kernel([be]):
                    return F.scaled_dot_product_attention(qt, ke, ve, is_causal=True)
            impls[name] = f
        try:
            import flashinfer

            qc, kc, vc = q.contiguous(), k.contiguous(), v.contiguous()
            impls["flashinfer_single_prefill"] = lambda: flashinfer.single_prefill_with_kv_cache(
                qc, kc, vc, causal=True)
        except Exception as exc:  # noqa: BLE001
            print(json.dumps({"n": n, "impl": "flashinfer_single_prefill", "error": str(exc)[:200]}), flush=True)
        ref = None
        for name, fn in impls.items():
            try:
                ms = timed(fn, iters)
                res = fn()
                torch.cuda.synchronize()
                if name == "prefillonly_tcgen05":
                    got = out.float()
                else:
                    r = res[0] if isinstance(res, tuple) else res
                    got = (r[0].transpose(0, 1) if r.dim() == 4 else r).reshape(n, HQ * D).float()
                if ref is None:
                    ref = got
                err = (got - ref).abs().max().item()
                print(json.dumps({"device": dev, "n": n, "impl": name, "ms": round(ms, 3),
                                  "tflops": round(flops / ms / 1e9, 1), "max_abs_diff_vs_ours": err}), flush=True)
            except Exception as exc:  # noqa: BLE001
                print(json.dumps({"n": n, "impl": name, "error": str(exc)[:200]}), flush=True)
        del qkv, out, qt, kt, vt, ke, ve
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [4096, 20000, 65536])

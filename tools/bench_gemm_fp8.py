"""CUDA-event timing of po_op_gemm_fp8 (E4M3 W8A8) next to po_op_gemm (bf16) at layer shapes (Llama-3.1-8B,
Qwen-2.5-32B). Inputs are reused across iterations (L2-warm for the smaller operands)."""
import ctypes, sys, json
import torch
sys.path.insert(0, ".")
from paper_2505_07203_b200 import _lib


def p(t): return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def timed(f, iters=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(iters): f()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def run(M, N, K):
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda") * K ** -0.5).to(torch.bfloat16)
    Aq = torch.empty(M, K, dtype=torch.uint8, device="cuda"); sa = torch.empty(M, device="cuda")
    Bq = torch.empty(N, K, dtype=torch.uint8, device="cuda"); sb = torch.empty(N, device="cuda")
    _lib.call("po_op_quantize_e4m3", p(A), K, M, K, p(Aq), K, p(sa), None)
    _lib.call("po_op_quantize_e4m3", p(B), K, N, K, p(Bq), K, p(sb), None)
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    f8 = lambda: _lib.call("po_op_gemm_fp8", p(Aq), K, p(sa), p(Bq), K, p(sb), p(out), N, None, 0, M, N, K,
                           _lib.EPI_BF16, None, 0, 0, None)
    bf = lambda: _lib.call("po_op_gemm", p(A), K, p(B), K, p(out), N, None, 0, M, N, K, _lib.EPI_BF16, None, 0, 0, None)
    q = lambda: _lib.call("po_op_quantize_e4m3", p(A), K, M, K, p(Aq), K, p(sa), None)
    t8, tb, tq = timed(f8), timed(bf), timed(q)
    fl = 2.0 * M * N * K
    print(json.dumps({"M": M, "N": N, "K": K, "fp8_ms": round(t8, 4), "fp8_tflops": round(fl / t8 / 1e9, 1),
                      "bf16_ms": round(tb, 4), "bf16_tflops": round(fl / tb / 1e9, 1),
                      "quantize_A_ms": round(tq, 4), "quantize_A_GBs": round(M * K * 3 / tq / 1e6, 1)}), flush=True)


if __name__ == "__main__":
    run(8192, 8192, 8192)
    run(8192, 28672, 4096)   # Llama gate/up chunk
    run(8192, 4096, 14336)   # Llama down chunk
    run(8192, 55296, 5120)   # Qwen-32B gate/up chunk
    run(8192, 5120, 27648)   # Qwen-32B down chunk
    run(160, 28672, 4096)    # prefix-hit gate/up (weight stream: half the bytes of bf16)
    run(160, 6144, 4096)     # prefix-hit QKV (split-K)

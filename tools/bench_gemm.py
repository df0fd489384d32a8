"""Quick CUDA-event timing of po_op_gemm vs torch.matmul (cuBLAS) at the Llama-3.1-8B layer shapes."""
import ctypes, sys, json
import torch
sys.path.insert(0, ".")
from paper_2505_07203_b200 import _lib

def p(t): return ctypes.c_void_p(t.data_ptr()) if t is not None else None

def run(M, N, K, epi=_lib.EPI_BF16, iters=20):
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda") * K ** -0.5).to(torch.bfloat16)
    ncols = N // 2 if epi == _lib.EPI_SILU_MUL else N
    out = torch.empty(M, ncols, dtype=torch.bfloat16, device="cuda")
    resid = torch.zeros(M, N, device="cuda") if epi == _lib.EPI_RESID_F32 else None
    f = lambda: _lib.call("po_op_gemm", p(A), K, p(B), K, p(out), ncols, p(resid), N, M, N, K, epi, None, 0, 0, None)
    for _ in range(3): f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(iters): f()
    e.record(); torch.cuda.synchronize()
    t = s.elapsed_time(e) / iters
    for _ in range(3): torch.matmul(A, B.T)
    s.record()
    for _ in range(iters): torch.matmul(A, B.T)
    e.record(); torch.cuda.synchronize()
    tc = s.elapsed_time(e) / iters
    fl = 2.0 * M * N * K
    print(json.dumps({"M": M, "N": N, "K": K, "epi": epi, "ms": round(t, 4), "tflops": round(fl / t / 1e9, 1),
                      "cublas_ms": round(tc, 4), "cublas_tflops": round(fl / tc / 1e9, 1)}), flush=True)

if __name__ == "__main__":
    run(8192, 8192, 8192)
    run(20000, 6144, 4096)
    run(20000, 4096, 4096, _lib.EPI_RESID_F32)
    run(8192, 28672, 4096, _lib.EPI_SILU_MUL)
    run(8192, 4096, 14336, _lib.EPI_RESID_F32)

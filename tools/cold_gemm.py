"""Cold-L2 device time of single po_op_gemm launches (a 400 MB read evicts L2 before each; a write-based flush would
leave dirty lines whose write-back competes with the kernel): python tools/cold_gemm.py"""
import ctypes, sys
import torch
sys.path.insert(0, ".")
from paper_2505_07203_b200 import _lib

SHAPES = [(160, 28672, 4096, 0), (16, 28672, 4096, 0), (160, 6144, 4096, 0), (160, 4096, 4096, 1), (160, 4096, 14336, 1)]

def main():
    flush = torch.ones(100 * 2**20, dtype=torch.float32, device="cuda")  # 400 MB, read to evict L2 (clean lines)
    p = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None
    for (M, N, K, epi) in SHAPES:
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        B = (torch.randn(N, K, device="cuda") * K ** -0.5).to(torch.bfloat16)
        out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        resid = torch.zeros(M, N, device="cuda")
        ts = []
        for it in range(6):
            flush.sum()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(True), torch.cuda.Event(True)
            s.record()
            _lib.call("po_op_gemm", p(A), K, p(B), K, p(out), N, p(resid), N, M, N, K, epi, None, 0, 0, None)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e) * 1e3)
        print(M, N, K, epi, "cold us", [round(x, 1) for x in ts[2:]], "weight GB/s", round(N * K * 2 / min(ts[2:]) / 1e3),
              flush=True)

if __name__ == "__main__":
    main()

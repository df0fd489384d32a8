#!/bin/bash
# ncu --set full on one FP8 (E4M3 W8A8) pair-GEMM launch at the Llama gate/up chunk shape (8192 x 28672 x 4096)
OUT=gpurun_out; mkdir -p $OUT
cat > /tmp/fp8_one.py <<'PY'
import ctypes, sys, torch
sys.path.insert(0, ".")
from paper_2505_07203_b200 import _lib
p = lambda t: ctypes.c_void_p(t.data_ptr())
M, N, K = 8192, 28672, 4096
A = torch.randn(M, K, device="cuda").to(torch.bfloat16); B = (torch.randn(N, K, device="cuda") * K ** -0.5).to(torch.bfloat16)
Aq = torch.empty(M, K, dtype=torch.uint8, device="cuda"); sa = torch.empty(M, device="cuda")
Bq = torch.empty(N, K, dtype=torch.uint8, device="cuda"); sb = torch.empty(N, device="cuda")
_lib.call("po_op_quantize_e4m3", p(A), K, M, K, p(Aq), K, p(sa), None)
_lib.call("po_op_quantize_e4m3", p(B), K, N, K, p(Bq), K, p(sb), None)
out = torch.empty(M, N // 2, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    _lib.call("po_op_gemm_fp8", p(Aq), K, p(sa), p(Bq), K, p(sb), p(out), N // 2, None, 0, M, N, K, _lib.EPI_SILU_MUL, None, 0, 0, None)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm2_kernel -s 1 -c 1 -o $OUT/fp8_gateup_full -f \
  python /tmp/fp8_one.py > $OUT/ncu_fp8.log 2>&1
ls -la $OUT/fp8_gateup_full.ncu-rep

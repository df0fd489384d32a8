"""Small invocations of every kernel for compute-sanitizer (memcheck / racecheck / synccheck)."""
import ctypes, sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2505_07203_b200 import _lib
from paper_2505_07203_b200.config import TINY
from paper_2505_07203_b200.engine import Engine

p = lambda t: ctypes.c_void_p(t.data_ptr())
# GEMM: 1-CTA (M<=128), pair (M>128), split-K, every epilogue
for M, N, K in ((100, 256, 256), (300, 512, 256), (160, 512, 2048)):
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    resid = torch.zeros(M, N, device="cuda")
    for epi in (0, 1, 2):
        _lib.call("po_op_gemm", p(A), K, p(B), K, p(out), N, p(resid), N, M, N, K, epi, None, 0, 0, None)
# attention: cold, prefix offset (split-KV + packed), odd group
for n, off, hq, hkv in ((300, 0, 4, 2), (600, 560, 8, 2), (300, 0, 5, 1)):
    ld = (hq + 2 * hkv) * 128
    qkv = torch.randn(n, ld, device="cuda").to(torch.bfloat16)
    out = torch.empty(n - off, hq * 128, dtype=torch.bfloat16, device="cuda")
    _lib.call("po_op_attention", p(qkv), ld, n, off, hq, hkv, p(out), hq * 128, None)
# engine: cold with admission, then prefix hits read straight from the pool (tile-aligned and straddling prefixes),
# for the tiny model (pair-GEMM epilogue admission) and a wider one (split-K reduce admission)
from paper_2505_07203_b200.config import ModelConfig
SMALL = ModelConfig("small", 2, 1024, 8, 2, 128, 2816, 4096)
for model in (TINY, SMALL):
    with Engine(model, seed=1, max_tokens=1024, chunk=256, pool_blocks=128) as e:
        t = np.random.default_rng(0).integers(0, 2**32, size=800, dtype=np.uint32)
        slots = list(range(800 // 16))
        e.prefill(t[:600], [1, 2], 0, slots[:37])
        e.prefill(t[:600], [1, 2], 512, slots[:37])
        e.prefill(t, [1, 2], 592, slots)  # straddling tile + suffix admission
# FP8: per-row quantisation, the W8A8 pair GEMM (full tiles, ragged M, split-K) with every epilogue, and an FP8 engine
from paper_2505_07203_b200.config import TINY_FP8
for M, N, K in ((300, 512, 256), (160, 512, 2048), (1, 256, 1024)):
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    Aq = torch.empty(M, K, dtype=torch.uint8, device="cuda"); sa = torch.empty(M, device="cuda")
    Bq = torch.empty(N, K, dtype=torch.uint8, device="cuda"); sb = torch.empty(N, device="cuda")
    _lib.call("po_op_quantize_e4m3", p(A), K, M, K, p(Aq), K, p(sa), None)
    _lib.call("po_op_quantize_e4m3", p(B), K, N, K, p(Bq), K, p(sb), None)
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    resid = torch.zeros(M, N, device="cuda")
    for epi in (0, 1, 2):
        _lib.call("po_op_gemm_fp8", p(Aq), K, p(sa), p(Bq), K, p(sb), p(out), N, p(resid), N, M, N, K, epi, None, 0, 0,
                  None)
with Engine(TINY_FP8, seed=1, max_tokens=1024, chunk=256, pool_blocks=64) as e:
    t = np.random.default_rng(1).integers(0, 2**32, size=700, dtype=np.uint32)
    slots = list(range(700 // 16))
    e.prefill(t, [1, 2], 0, slots)
    e.prefill(t, [1, 2], 512, slots)
# round 2: multi-CTA LM head (allowed list > 256 rows); an engine whose MLP runs 512-row pieces (fused MLP launch
# under PO_FUSED_MLP=1); prefix hits through the stream-K kernel (default: gate/up; PO_SK=1: every epilogue)
with Engine(TINY, seed=1, max_tokens=2048, chunk=1024, pool_blocks=128) as e:
    t = np.random.default_rng(2).integers(0, 2**32, size=1300, dtype=np.uint32)
    slots = list(range(1300 // 16))
    e.prefill(t, list(range(0, 32000, 7)), 0, slots)
    e.prefill(t, [1, 2], 1296 // 16 * 16 - 160, slots)
torch.cuda.synchronize()
print("sanitize workload done")

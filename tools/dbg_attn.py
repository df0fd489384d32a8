import ctypes, sys, torch
sys.path.insert(0, ".")
from paper_2505_07203_b200 import _lib
n, hq, hkv = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
ld = (hq + 2 * hkv) * 128
qkv = torch.randn(n, ld, device="cuda").to(torch.bfloat16)
out = torch.zeros(n, hq * 128, dtype=torch.bfloat16, device="cuda")
rc = _lib.load().po_op_attention(qkv.data_ptr(), ld, n, 0, hq, hkv, out.data_ptr(), hq * 128, None)
print("rc", rc); torch.cuda.synchronize(); print("done", out.float().abs().sum().item())

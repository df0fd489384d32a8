"""Hit-shape attention (20,000 keys, 160 queries, Llama-3.1-8B heads) through po_op_attention: per-launch time of 1 / 10 /
200 back-to-back launches (split-KV + combine) with the SM clock read after each loop."""
import ctypes, sys, torch, subprocess
sys.path.insert(0, ".")
from paper_2505_07203_b200 import _lib
n, off = 20000, 19840
hq, hkv = 32, 8
ld = (hq + 2 * hkv) * 128
qkv = torch.randn(n, ld, device="cuda").to(torch.bfloat16)
out = torch.empty(n - off, hq * 128, dtype=torch.bfloat16, device="cuda")
ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
f = lambda: _lib.call("po_op_attention", ctypes.c_void_p(qkv.data_ptr()), ld, n, off, hq, hkv, ctypes.c_void_p(out.data_ptr()), hq * 128, None)
for _ in range(5): f()
torch.cuda.synchronize()
for it in (1, 10, 200):
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(it): f()
    e.record(); torch.cuda.synchronize()
    c = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip()
    print(it, "launches: us per launch", round(s.elapsed_time(e) / it * 1e3, 1), "clock after", c)

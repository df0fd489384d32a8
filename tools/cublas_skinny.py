import torch
flush = torch.ones(100 * 2**20, dtype=torch.float32, device="cuda")  # 400 MB, read to evict L2 (clean lines)
for M in (16, 160):
    W = torch.randn(28672, 4096, device="cuda").to(torch.bfloat16)
    x = torch.randn(M, 4096, device="cuda").to(torch.bfloat16)
    ts = []
    for it in range(6):
        flush.sum(); torch.cuda.synchronize()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); y = torch.mm(x, W.T); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    print("cublas M", M, "cold us", [round(t, 1) for t in ts[2:]], "GB/s", round(W.numel() * 2 / min(ts[2:]) / 1e3))

"""Per-kernel-class CUDA-event breakdown of cold and prefix-hit Llama-3.1-8B forwards."""
import sys, json
import numpy as np
sys.path.insert(0, ".")
from paper_2505_07203_b200.engine import Engine
from paper_2505_07203_b200.config import LLAMA_3_1_8B as M

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
e = Engine(M, seed=0, max_tokens=max(n, 20480), pool_blocks=2048)
toks = np.random.default_rng([0, 0, 0]).integers(0, 2**32, size=n, dtype=np.uint32)
nb = n // 16
slots = list(range(nb))
e.prefill(toks, [9642, 2822], 0, slots)
for nc in (0, (n - 160) // 16 * 16):
    ids = slots[: nc // 16] + [-1] * (nb - nc // 16)
    for _ in range(2):
        e.prefill(toks, [9642, 2822], nc, ids)
    e.profile_begin()
    r = e.prefill(toks, [9642, 2822], nc, ids)
    prof = e.profile_end()
    tot = sum(v[0] for v in prof.values())
    print(json.dumps({"n": n, "n_cached": nc, "service_ms": round(r.service_s * 1e3, 3), "sum_kernel_ms": round(tot, 3),
                      "launches": e.last_launches,
                      "classes": {k: [round(v[0], 3), v[1]] for k, v in prof.items() if v[1]}}), flush=True)

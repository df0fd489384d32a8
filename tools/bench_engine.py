"""Quick end-to-end timing of Engine.prefill on Llama-3.1-8B shapes (random-init bf16)."""
import sys, time, json
import numpy as np
sys.path.insert(0, ".")
from paper_2505_07203_b200.engine import Engine
from paper_2505_07203_b200.config import LLAMA_3_1_8B as M

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
t0 = time.time()
e = Engine(M, seed=0, max_tokens=max(n, 20480), chunk=chunk, pool_blocks=2048)
print("init s", round(time.time() - t0, 2), "weights GB", e.weight_bytes / 1e9, "arena GB", e.arena_bytes / 1e9, flush=True)
toks = np.random.default_rng([0, 0, 0]).integers(0, 2**32, size=n, dtype=np.uint32)
for i in range(4):
    r = e.prefill(toks, [9642, 2822], pool_block_ids=list(range(min(n // 16, 2048))) if i == 0 else None)
    fl = M.request_flops(n)
    print(json.dumps({"n": n, "service_s": round(r.service_s, 4), "tok_s": round(n / r.service_s),
                      "tflops": round(fl / r.service_s / 1e12, 1), "argmax": r.index, "probs": r.probs.tolist()}), flush=True)
nc = (min(n // 16, 2048) * 16) - 16 * 10
if nc > 0:
    r = e.prefill(toks, [9642, 2822], n_cached=nc, pool_block_ids=list(range(nc // 16)))
    print(json.dumps({"n": n, "n_cached": nc, "service_s": round(r.service_s, 4), "probs": r.probs.tolist()}))

import sys; sys.path.insert(0, ".")
import numpy as np
from paper_2505_07203_b200.config import QWEN_2_5_32B_FP8, QWEN_2_5_32B, TINY_FP8
from paper_2505_07203_b200.engine import Engine
Y = [9642, 2822]
for M, n in ((QWEN_2_5_32B_FP8, 10000), (QWEN_2_5_32B, 10000), (QWEN_2_5_32B_FP8, 2048)):
    toks = np.random.default_rng([5, 0, 0]).integers(0, 2**32, size=n, dtype=np.uint32)
    with Engine(M, seed=0, max_tokens=n, pool_blocks=n // 16 + 8) as e:
        slots = list(range(n // 16))
        cold = e.prefill(toks, Y, 0, slots)
        hits = [e.prefill(toks, Y, nc, slots).logits for nc in (n - 160, n // 2 // 16 * 16, 16)]
        cold2 = e.prefill(toks, Y)
    print(M.name, n, "cold", cold.logits, "cold2", cold2.logits, "hits", hits, flush=True)

"""One warm prefix-hit forward (19,840 cached + 160 miss tokens) for kernel-level profiling."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2505_07203_b200.engine import Engine
from paper_2505_07203_b200.config import LLAMA_3_1_8B as M
n = 20000
e = Engine(M, seed=0, max_tokens=20480, pool_blocks=1400)
toks = np.random.default_rng([0, 0, 0]).integers(0, 2**32, size=n, dtype=np.uint32)
slots = list(range(n // 16))
e.prefill(toks, [9642, 2822], 0, slots)
nc = (n - 160) // 16 * 16
for _ in range(3):
    r = e.prefill(toks, [9642, 2822], nc, slots)
print("hit service ms", r.service_s * 1e3)

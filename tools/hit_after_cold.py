"""Prefix-hit service time right after a cold 20k forward vs after other hits (the serving mix interleaves them)."""
import statistics
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2505_07203_b200.engine import Engine
from paper_2505_07203_b200.config import LLAMA_3_1_8B as M
n = 20000
e = Engine(M, seed=0, max_tokens=20480, pool_blocks=4096)
nb = n // 16
nc = (n - 160) // 16 * 16
after_cold, after_hit = [], []
for u in range(6):
    toks = np.random.default_rng([u, 0, 0]).integers(0, 2**32, size=n, dtype=np.uint32)
    slots = [(u % 2) * nb + b for b in range(nb)]
    e.prefill(toks, [9642, 2822], 0, slots)
    after_cold.append(e.prefill(toks, [9642, 2822], nc, slots).service_s * 1e3)
    after_hit.append(e.prefill(toks, [9642, 2822], nc, slots).service_s * 1e3)
print("hit right after cold ms", [round(x, 2) for x in after_cold], "median", round(statistics.median(after_cold), 2))
print("hit after a hit ms", [round(x, 2) for x in after_hit], "median", round(statistics.median(after_hit), 2))
# recovery curve: ten hits back to back after a cold forward
toks = np.random.default_rng([9, 0, 0]).integers(0, 2**32, size=n, dtype=np.uint32)
slots = list(range(nb))
e.prefill(toks, [9642, 2822], 0, slots)
curve = [e.prefill(toks, [9642, 2822], nc, slots).service_s * 1e3 for _ in range(12)]
print("hits after a cold, in order ms", [round(x, 2) for x in curve])

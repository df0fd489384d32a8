"""Warm prefix-hit forwards (19,840 cached + 160 miss tokens) for kernel-level profiling and A/B timing:
prints the median service time of 20 forwards after 5 untimed ones (python tools/hit_once.py [n_forwards])."""
import statistics
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2505_07203_b200.engine import Engine
from paper_2505_07203_b200.config import LLAMA_3_1_8B as M
n = 20000
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
e = Engine(M, seed=0, max_tokens=20480, pool_blocks=1400)
toks = np.random.default_rng([0, 0, 0]).integers(0, 2**32, size=n, dtype=np.uint32)
slots = list(range(n // 16))
e.prefill(toks, [9642, 2822], 0, slots)
nc = (n - 160) // 16 * 16
for _ in range(5 if reps > 1 else 0):  # clocks settle under back-to-back load first
    e.prefill(toks, [9642, 2822], nc, slots)
ts = [e.prefill(toks, [9642, 2822], nc, slots).service_s * 1e3 for _ in range(reps)]
print("hit service ms median", round(statistics.median(ts), 3), "min", round(min(ts), 3))

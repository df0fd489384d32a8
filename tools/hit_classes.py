"""Per-kernel-class device time of warm prefix-hit forwards (19,840 cached + 160 miss tokens), CUDA events around
every class on the engine stream (events break the PDL overlap, so the sum exceeds the plain forward time; compare
shares): python tools/hit_classes.py [n_forwards]"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2505_07203_b200.config import LLAMA_3_1_8B as M  # noqa: E402
from paper_2505_07203_b200.engine import Engine  # noqa: E402

n = 20000
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
e = Engine(M, seed=0, max_tokens=20480, pool_blocks=1400)
toks = np.random.default_rng([0, 0, 0]).integers(0, 2 ** 32, size=n, dtype=np.uint32)
slots = list(range(n // 16))
e.prefill(toks, [9642, 2822], 0, slots)
nc = (n - 160) // 16 * 16
for _ in range(5):
    e.prefill(toks, [9642, 2822], nc, slots)
e.profile_begin()
for _ in range(reps):
    e.prefill(toks, [9642, 2822], nc, slots)
prof = e.profile_end()
tot = sum(v[0] for v in prof.values())
for k, (ms, cnt) in prof.items():
    if cnt:
        print(f"{k:20s} {ms / reps:8.3f} ms/forward  {cnt // reps:4d} launches  share {ms / tot:.3f}")
print(f"sum {tot / reps:.3f} ms/forward")

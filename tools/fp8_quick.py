"""Cold-request service time of the FP8 presets at one length each (quick A/B of FP8 kernel changes):
python tools/fp8_quick.py -> llama-3.1-8b-fp8 20k and qwen-2.5-32b-fp8 10k, median of 3 after 2 warm-ups."""
import statistics
import sys
from dataclasses import replace

import numpy as np

sys.path.insert(0, ".")
from paper_2505_07203_b200.config import LLAMA_3_1_8B, QWEN_2_5_32B_FP8  # noqa: E402
from paper_2505_07203_b200.engine import Engine  # noqa: E402

for M, n in ((replace(LLAMA_3_1_8B, name="llama-3.1-8b-fp8", weight_fp8=True), 20_000), (QWEN_2_5_32B_FP8, 10_000)):
    toks = np.random.default_rng([3, 0, 0]).integers(0, 2 ** 32, size=n, dtype=np.uint32)
    with Engine(M, seed=0, max_tokens=n + 512, pool_blocks=64) as e:
        for _ in range(2):
            e.prefill(toks, [9642, 2822])
        ts = [e.prefill(toks, [9642, 2822]).service_s for _ in range(3)]
    t = statistics.median(ts)
    print(f"{M.name} n={n}: {t * 1e3:.1f} ms, {n / t:.0f} tok/s, {M.request_flops(n) / t / 1e12:.0f} TFLOP/s",
          flush=True)

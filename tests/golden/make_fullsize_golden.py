"""Oracle fixtures at the TARGET shapes (Llama-3.1-8B dims, 2 layers) for tests/test_gpu_parity_fullsize.py.

    python tests/golden/make_fullsize_golden.py          # ~10 min on 8 cores, ~15 GB RAM

Runs the CPU oracle (oracle/llama_ref.py: bf16-faithful float64 restatement of the layer forward,
ps/numerics.py:132-171 + the stated Llama definitions) on Llama-3.1-8B layer shapes (h=4096, 32 q / 8 kv heads of 128,
I=14336, vocab 128,256, llama3 RoPE) with the first two layers of the engine's counter-hash weights (seed 0). The GPU
box has no time for an f64 20k-token forward, so the results are committed as tests/golden/fullsize_golden.json:
logits, probs, argmax and the top-2 margin over the allowed ids, per case. Nothing here runs at test time.

Cases (BASELINE configs[1] shapes):
  cold_20000  one 20,000-token request (79 pair row tiles of 256 rows, 3 MLP chunks of 8192, 157 key tiles)
  cold_8300   8,300 tokens: crosses the 8,192-row MLP chunk boundary by 108 rows
The prefix-hit test (19,840 cached + 160) reuses cold_20000: cached rows only serve as keys, so a hit's answer is the
cold forward's.
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from dataclasses import replace
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import llama_ref  # noqa: E402
from paper_2505_07203_b200.config import LLAMA_3_1_8B  # noqa: E402

OUT = Path(__file__).with_name("fullsize_golden.json")
SEED = 0
LAYERS = 2
ALLOWED = [9642, 2822, 0, 1, 1000, 50_000, 100_000, 128_255]  # "Yes", "No" + six spread ids
CASES = {"cold_20000": (101, 20_000), "cold_8300": (102, 8_300)}


def tokens_for(seed: int, n: int) -> np.ndarray:
    # same stream construction as the reference workloads (ps/workload.py:113-115) and tests/test_gpu_engine.py
    return np.random.default_rng([seed, 0, 0]).integers(0, 2 ** 32, size=n, dtype=np.uint32)


def main():
    model = replace(LLAMA_3_1_8B, num_layers=LAYERS)
    cfg = llama_ref.Cfg.from_model(model)
    t0 = time.time()
    w = llama_ref.make_weights(cfg, SEED, lazy_vocab=True)
    print(f"weights {time.time() - t0:.1f} s", flush=True)
    out = {"model": "llama-3.1-8b", "num_layers": LAYERS, "seed": SEED, "allowed": ALLOWED,
           "generator": "tests/golden/make_fullsize_golden.py (oracle/llama_ref.llama_forward, float64, bf16 storage)",
           "cases": {}}
    for name, (tseed, n) in CASES.items():
        toks = tokens_for(tseed, n)
        t1 = time.time()
        logits, probs, am = llama_ref.llama_forward(cfg, w, toks, ALLOWED)
        srt = np.sort(logits)[::-1]
        out["cases"][name] = {
            "token_seed": tseed, "n": n, "tokens_sha256": hashlib.sha256(toks.tobytes()).hexdigest(),
            "logits": logits.tolist(), "probs": probs.tolist(), "argmax": am, "top2_margin": float(srt[0] - srt[1]),
            "oracle_seconds": round(time.time() - t1, 1)}
        print(name, out["cases"][name], flush=True)
        OUT.write_text(json.dumps(out, indent=1))
    print(f"wrote {OUT} in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()

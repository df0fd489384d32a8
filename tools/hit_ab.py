"""A/B of environment switches on the warm prefix-hit forward (19,840 cached + 160 miss tokens, Llama-3.1-8B):
each setting runs in its own process (the switches are read once per process); median device service time of 30
back-to-back hits, three alternating rounds so clock drift hits every setting alike.
python tools/hit_ab.py 'PO_ATTN_L2PF=0' 'PO_ATTN_L2PF=1' 'PO_ATTN_L2PF=2'"""
import json
import os
import subprocess
import sys

CHILD = r'''
import sys, json, numpy as np
sys.path.insert(0, ".")
from paper_2505_07203_b200.config import LLAMA_3_1_8B as M
from paper_2505_07203_b200.engine import Engine
n = 20000
e = Engine(M, seed=0, max_tokens=20480, pool_blocks=1400)
toks = np.random.default_rng([7, 1, 0]).integers(0, 2 ** 32, size=n, dtype=np.uint32)
slots = list(range(n // 16))
r0 = e.prefill(toks, [9642, 2822], 0, slots)
nc = (n - 160) // 16 * 16
for _ in range(8):
    e.prefill(toks, [9642, 2822], nc, slots)
ts = []
for _ in range(30):
    r = e.prefill(toks, [9642, 2822], nc, slots)
    ts.append(r.service_s)
ts.sort()
print(json.dumps({"med_ms": ts[15] * 1e3, "min_ms": ts[0] * 1e3, "index": int(r.index), "cold_index": int(r0.index),
                  "logits": [float(x) for x in r.logits]}))
'''

settings = sys.argv[1:] or ["PO_ATTN_L2PF=0", "PO_ATTN_L2PF=2"]
res = {s: [] for s in settings}
for rnd in range(3):
    for s in settings:
        env = dict(os.environ)
        for kv in s.split(","):
            if kv:
                k, v = kv.split("=")
                env[k] = v
        out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=600)
        if out.returncode:
            print(s, "FAILED", out.stderr[-2000:])
            continue
        d = json.loads(out.stdout.strip().splitlines()[-1])
        res[s].append(d)
        print(f"round {rnd} {s:40s} med {d['med_ms']:.3f} ms  min {d['min_ms']:.3f}  idx {d['index']} "
              f"logits {d['logits']}", flush=True)
for s, ds in res.items():
    if ds:
        print(f"{s:40s} median-of-medians {sorted(x['med_ms'] for x in ds)[len(ds) // 2]:.3f} ms")

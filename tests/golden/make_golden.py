"""Generate golden fixtures by running the REFERENCE (arxiv 2505.07203 `prefillsim`) in this container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/reference_golden.json. The reference is imported read-only from /root/reference; it is
not available on the GPU box, so the tests read only the committed JSON. Everything is seeded.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

from prefillsim import cache as rcache  # noqa: E402
from prefillsim import costs as rcosts  # noqa: E402
from prefillsim import geometry as rgeom  # noqa: E402
from prefillsim import jct as rjct  # noqa: E402
from prefillsim import numerics as rnum  # noqa: E402
from prefillsim import presets as rpresets  # noqa: E402
from prefillsim import scheduling as rsched  # noqa: E402
from prefillsim import sim as rsim  # noqa: E402
from prefillsim import workload as rwl  # noqa: E402

OUT = Path(__file__).with_name("reference_golden.json")


def hx(chain):
    return [d.hex() for d in chain]


def gen_block_chains():
    cases = []
    for seed, n, bt in [(0, 0, 16), (1, 15, 16), (2, 16, 16), (3, 100, 16), (4, 1000, 16), (5, 257, 8), (6, 64, 1)]:
        toks = np.random.default_rng([seed, 77]).integers(0, 2 ** 32, size=n, dtype=np.uint32)
        cases.append({"seed": seed, "n": n, "bt": bt, "chain": hx(rcache.block_chain(toks, bt))})
    return cases


def chain_universe(rng, n_prefixes=6, max_blocks=24):
    """Random sequences built from shared prefixes so inserts overlap."""
    bases = [rng.integers(0, 2 ** 32, size=16 * max_blocks, dtype=np.uint32) for _ in range(n_prefixes)]
    seqs = []
    for _ in range(40):
        b = bases[int(rng.integers(0, n_prefixes))]
        cut = int(rng.integers(1, max_blocks + 1)) * 16
        tail = rng.integers(0, 2 ** 32, size=int(rng.integers(0, 64)), dtype=np.uint32)
        seqs.append(np.concatenate([b[:cut], tail]))
    return seqs


def gen_cache_ops():
    rng = np.random.default_rng(2024)
    seqs = chain_universe(rng)
    chains = [rcache.block_chain(s, 16) for s in seqs]
    cache = rcache.PrefixCache(rcache.CacheConfig(capacity_tokens=16 * 48, block_tokens=16))
    ops = []
    now = 0.0
    for step in range(400):
        now += float(rng.integers(0, 3))  # equal timestamps exercise the ins_order tie-break
        k = int(rng.integers(0, len(chains)))
        kind = int(rng.integers(0, 10))
        if kind < 5:
            out = cache.insert_chain(chains[k], now)
            ops.append({"op": "insert", "seq": k, "now": now, "out": out})
        elif kind < 9:
            ops.append({"op": "match", "seq": k, "out": cache.match_chain(chains[k])})
        else:
            need = int(rng.integers(0, 20)) * 16
            try:
                out = cache.evict_to(need, protect=chains[k])
            except rcache.EvictionShortfall as e:
                out = -1 - e.freed_tokens
            ops.append({"op": "evict_to", "seq": k, "need": need, "out": out})
        ops[-1]["used"] = cache.used_tokens
        ops[-1]["resident"] = sorted(d.hex() for d in cache._blocks)[:4] if step % 50 == 0 else None
    return {"seqs": [s.tolist() for s in seqs], "capacity_tokens": 16 * 48, "bt": 16, "ops": ops,
            "final_resident": sorted(d.hex() for d in cache._blocks)}


class _Req:
    def __init__(self, rid, n, tokens, user=0):
        self.id, self.user_id, self.n_input, self.tokens = rid, user, n, tokens


def gen_scheduler_cases():
    rng = np.random.default_rng(11)
    seqs = chain_universe(rng, n_prefixes=4, max_blocks=16)
    cases = []
    for c in range(60):
        cache = rcache.PrefixCache(rcache.CacheConfig(capacity_tokens=16 * 40, block_tokens=16))
        for k in rng.integers(0, len(seqs), size=int(rng.integers(0, 6))):
            cache.insert(seqs[int(k)], now=float(rng.uniform(0, 5)))
        q = []
        for i in rng.choice(len(seqs), size=int(rng.integers(1, 12)), replace=False):
            s = seqs[int(i)]
            wr = rsched.WaitingRequest(request=_Req(int(i), len(s), s), arrival=float(rng.integers(0, 20)) / 2,
                                       frozen_jct=float(rng.integers(0, 2000)),
                                       chain=rcache.block_chain(s, 16))
            q.append(wr)
        now = 20.0
        picks = {}
        for name, pol in [("fifo", rsched.Policy.fifo()), ("srjf", rsched.Policy.srjf_static()),
                          ("cal0", rsched.Policy.srjf_calibrated(lam=0.0)),
                          ("cal05", rsched.Policy.srjf_calibrated(lam=0.5)),
                          ("cal500", rsched.Policy.srjf_calibrated(lam=500.0)),
                          ("calprof", rsched.Policy.srjf_calibrated(lam=0.01, scoring="profile"))]:
            prof = rjct.JctProfile(2e-5, -1.5e-5, 0.01, 1.0)
            order = []
            pending = list(q)
            while pending:
                w = rsched.schedule_next(pending, cache, prof, pol, now)
                order.append(w.request.id)
                pending.remove(w)
            picks[name] = order
        cases.append({
            "inserted_state": [d.hex() for d in cache._blocks],
            "queue": [{"id": w.request.id, "n_input": w.request.n_input, "arrival": w.arrival,
                       "frozen_jct": w.frozen_jct, "n_cached": cache.match_chain(w.chain)} for w in q],
            "now": now, "orders": picks})
    return {"seqs": [s.tolist() for s in seqs], "cases": cases}


def small_post_rec(seed, users=6, per_user=12):
    spec_lengths = rwl.post_rec_profile_lengths(seed)[:users]
    reqs = []
    for u, plen in enumerate(spec_lengths):
        plen = plen // 8  # keep the fixture small: ~1.4k-2.1k token profiles
        for _ in range(per_user):
            reqs.append(rwl.Request(id=len(reqs), user_id=u, arrival=0.0, profile_len=plen,
                                    total_len=plen + rwl.POST_REC_SUFFIX_TOKENS, seed=seed))
    return rwl.Trace(name="post-rec-small", seed=seed, requests=tuple(reqs))


def gen_sim_runs():
    geom = rpresets.load_model("llama-3.1-8b")
    gpu = rpresets.load_gpu("l4")
    params = rcosts.CostParams.derive(geom, gpu)
    variant = rcosts.EngineVariant.prefill_only_hybrid()
    base = small_post_rec(3)
    runs = []
    for policy_name, policy in [("fifo", rsched.Policy.fifo()), ("srjf", rsched.Policy.srjf_static()),
                                ("srjf-calibrated", rsched.Policy.srjf_calibrated())]:
        for n_inst in (1, 2):
            for rate in (2.0, 8.0):
                trace = rwl.poisson_arrivals(base, rate, seed=5, keep_sessions=True)
                cfg = rsim.SimConfig(geom=geom, gpu=gpu, cost_params=params, variant=variant, policy=policy,
                                     num_instances=n_inst, cache_capacity_tokens=16 * 300)
                rep = rsim.run(trace, cfg)
                runs.append({"policy": policy_name, "instances": n_inst, "rate": rate,
                             "records": [[r.id, r.instance, r.start, r.completion, r.n_cached] for r in rep.records],
                             "mean": rep.mean_latency, "p99": rep.p99_latency, "throughput": rep.throughput,
                             "hit_requests": rep.cache_hit_requests, "hit_tokens": rep.cache_hit_tokens})
    return {"c_linear": params.c_linear, "c_attn": params.c_attn, "c_fixed": params.c_fixed,
            "capacity_tokens": 16 * 300, "trace_seed": 3, "users": 6, "per_user": 12, "arrival_seed": 5,
            "runs": runs}


def gen_workload():
    pr = rwl.gen_post_recommendation(0)
    cr = rwl.gen_credit_verification(0)
    arr = rwl.poisson_arrivals(pr, 2.5, seed=1, keep_sessions=True)
    arr2 = rwl.poisson_arrivals(cr, 0.7, seed=2, keep_sessions=False)
    r0 = pr.requests[51]
    return {
        "post_rec_profile_lengths": rwl.post_rec_profile_lengths(0),
        "credit_lengths": rwl.credit_lengths(0),
        "post_rec_tokens_req51_head": r0.tokens[:8].tolist(),
        "post_rec_tokens_req51_suffix": r0.suffix_tokens[:4].tolist(),
        "post_rec_req51_chain_sha256": hashlib.sha256(b"".join(r0.digest_chain(16, {}))).hexdigest(),
        "poisson_keep": [[r.id, r.arrival] for r in arr.requests[:60]],
        "poisson_interleave": [[r.id, r.arrival] for r in arr2.requests],
    }


def gen_worked_example():
    trace, cap = rwl.worked_example()
    out = {}
    geom = rpresets.load_model("llama-3.1-8b")
    gpu = rpresets.load_gpu("l4")
    params = rcosts.CostParams.derive(geom, gpu)
    for name, pol in [("fifo", rsched.Policy.fifo()), ("srjf", rsched.Policy.srjf_static()),
                      ("srjf-calibrated", rsched.Policy.srjf_calibrated())]:
        cfg = rsim.SimConfig(geom=geom, gpu=gpu, cost_params=params,
                             variant=rcosts.EngineVariant.prefill_only_hybrid(), policy=pol,
                             cache_capacity_tokens=cap)
        rep = rsim.run(trace, cfg)
        order = [r.id for r in sorted(rep.records, key=lambda r: r.start)]
        out[name] = {"order": order, "hits": rep.cache_hit_requests}
    return out


def gen_numerics():
    params = rnum.ToyBlockParams.random(42, hidden=16, intermediate=64)
    x = rnum.random_input(42, n=64, hidden=16)
    out = rnum.block_forward_full(params, x, rnum.ScratchTracker())
    cases = []
    rng = np.random.default_rng(99)
    for case in range(6):
        h = int(rng.integers(2, 24))
        inter = h * int(rng.integers(1, 5))
        n = int(rng.integers(1, 80))
        p = rnum.ToyBlockParams.random(case, h, inter)
        xi = rnum.random_input(case, n, h)
        ft, ht = rnum.ScratchTracker(), rnum.ScratchTracker()
        full = rnum.block_forward_full(p, xi, ft)
        hyb = rnum.block_forward_hybrid(p, xi.copy(), max(1, n // 3), ht, prealloc=True, inplace=True)
        cases.append({"case": case, "hidden": h, "inter": inter, "n": n, "chunk": max(1, n // 3),
                      "full_sha256": hashlib.sha256(np.round(full, 6).tobytes()).hexdigest(),
                      "full_first_row": full[0].tolist(), "peak_full": ft.peak, "peak_hybrid": ht.peak,
                      "max_abs_diff_hybrid": float(np.abs(full - hyb).max())})
    return {"seed42_sha256": hashlib.sha256(np.round(out, 6).tobytes()).hexdigest(), "seed42_out": out.tolist(),
            "cases": cases}


def gen_geometry_jct():
    geom = rpresets.load_model("llama-3.1-8b")
    gpu = rpresets.load_gpu("l4")
    params = rcosts.CostParams.derive(geom, gpu)
    variant = rcosts.EngineVariant.prefill_only_hybrid()
    mil = rcosts.variant_mil(variant, geom, gpu)
    samples = rjct.generate_samples(lambda n, nc: rcosts.execute_time(variant, geom, gpu, params, n, nc),
                                    max_input=min(mil, 60_000))
    prof = rjct.fit(samples)
    return {
        "kv_bytes_per_token": list(rgeom.kv_bytes_per_token(geom)),
        "linear_flops_per_token": rcosts.linear_flops_per_token(geom),
        "attn_flops_per_pair": rcosts.attn_flops_per_pair(geom),
        "grid_fit": [prof.coef_input, prof.coef_cached, prof.intercept, prof.fit_r2],
        "proxy_miss_14000_11000": rjct.proxy_miss(14000, 11000),
        "execute_time_20000_0": rcosts.execute_time(variant, geom, gpu, params, 20000, 0),
        "execute_time_20000_19840": rcosts.execute_time(variant, geom, gpu, params, 20000, 19840),
        "l4_hybrid_mil": mil,
    }


def main():
    golden = {
        "generated_from": "/root/reference/pkg/src/prefillsim (read-only), by tests/golden/make_golden.py",
        "block_chains": gen_block_chains(),
        "cache_ops": gen_cache_ops(),
        "scheduler": gen_scheduler_cases(),
        "sim_runs": gen_sim_runs(),
        "workload": gen_workload(),
        "worked_example": gen_worked_example(),
        "numerics": gen_numerics(),
        "geometry_jct": gen_geometry_jct(),
    }
    OUT.write_text(json.dumps(golden, separators=(",", ":")) + "\n")
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB)")


if __name__ == "__main__":
    main()

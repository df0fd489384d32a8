"""The wall-clock Server driving a real GPU Engine (ps/sim.py:211-269 contract).

About fifty post-recommendation requests (shared user profiles, so most are prefix hits served from the pool) go
through `serving.Server` on the tiny model. The scheduling order is checked against the oracle's schedule_next in
lock step (same queue, same cache evolution), every request completes with a result, and sampled answers (cold and
prefix-hit) equal the CPU oracle's.
"""

import threading
import time

import numpy as np
import pytest

from oracle import llama_ref, sched_ref
from paper_2505_07203_b200 import workload as wl
from paper_2505_07203_b200.config import TINY
from paper_2505_07203_b200.engine import Engine
from paper_2505_07203_b200.scheduling import Policy
from paper_2505_07203_b200.serving import Server, replay

pytestmark = pytest.mark.gpu

YES_NO = [9642, 2822]


def trace():
    spec = wl.PostRecSpec(users=5, requests_per_user=10, profile_mean=1500, profile_std=200, profile_min=1100,
                          profile_max=1900, suffix_tokens=100)
    return wl.gen_post_recommendation(11, spec)


@pytest.fixture(scope="module")
def engine():
    with Engine(TINY, seed=42, max_tokens=4096, chunk=1024, pool_blocks=2048) as e:
        yield e


def test_server_on_gpu_matches_oracle_order_and_answers(engine):
    gate = threading.Event()
    orig = engine.prefill
    seen = {}

    def gated(tokens, allowed, n_cached=0, pool_block_ids=None):
        gate.wait()
        res = orig(tokens, allowed, n_cached, pool_block_ids)
        seen[len(seen)] = (np.asarray(tokens).copy(), n_cached, res)
        return res

    engine.prefill = gated
    srv = Server([engine], Policy.srjf_calibrated(lam=0.0))
    try:
        tr = trace()
        futs = [srv.submit(r, YES_NO) for r in tr.requests]
        time.sleep(0.3)
        gate.set()
        results = [f.result(timeout=120) for f in futs]
    finally:
        srv.close()
        engine.prefill = orig
    assert len(results) == len(tr.requests) == 50
    assert all(r.token in YES_NO for r in results)
    order = [r.id for r in sorted(srv.records, key=lambda r: r.start)]
    # lock-step shadow: the oracle picks from the same queue with the same cache evolution
    cache = sched_ref.PrefixCache(engine.capacity_tokens)
    pending = [dict(id=r.id, n_input=r.n_input, arrival=0.0, frozen_jct=0.0, chain=r.digest_chain(16, {}))
               for r in tr.requests]
    first = next(p for p in pending if p["id"] == order[0])
    expected = [first["id"]]
    pending.remove(first)
    cache.insert_chain(first["chain"], 1.0)
    t = 2.0
    while pending:
        w = sched_ref.schedule_next(pending, cache, "cal", t, lam=0.0)
        expected.append(w["id"])
        pending.remove(w)
        cache.insert_chain(w["chain"], t)
        t += 1.0
    assert order == expected
    hits = [v for v in seen.values() if v[1] > 0]
    assert len(hits) >= 40  # every user's later requests reuse its cached profile
    # sampled answers against the CPU oracle: the first cold request and three prefix hits
    cfg = llama_ref.Cfg.from_model(TINY)
    w = llama_ref.make_weights(cfg, 42)
    colds = [v for v in seen.values() if v[1] == 0]
    for toks, n_cached, res in colds[:1] + hits[:3]:
        logits, _, am = llama_ref.llama_forward(cfg, w, toks, YES_NO)
        assert np.abs(res.logits - logits).max() <= 1e-2 + 5e-3 * np.abs(logits).max()
        assert res.index == am


def test_server_replay_on_gpu_in_real_time(engine):
    srv = Server([engine], Policy.srjf_calibrated())
    try:
        rep = replay(srv, wl.poisson_arrivals(trace(), 200.0, seed=2), YES_NO)
    finally:
        srv.close()
    assert rep.served == 50 and rep.cache_hit_requests >= 40
    assert rep.p99_latency > 0 and all(r.completion >= r.start >= r.arrival for r in rep.records)

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


@pytest.mark.parametrize("lookahead", [False, True])
def test_server_on_gpu_matches_oracle_order_and_answers(engine, lookahead):
    """lookahead=False decides when the engine frees up; lookahead=True (prefill_submit / prefill_wait, two
    forwards in flight) decides one request ahead. With every request queued before the first decision both take
    the oracle's decisions."""
    gate = threading.Event()
    orig_submit, orig_wait = engine.prefill_submit, engine.prefill_wait
    seen = {}
    pending_toks = {}

    def gated_submit(tokens, allowed, n_cached=0, pool_block_ids=None, stream=None):
        gate.wait()
        t = orig_submit(tokens, allowed, n_cached, pool_block_ids, stream)
        pending_toks[t.id] = (np.asarray(tokens).copy(), n_cached)
        return t

    def recording_wait(ticket):
        res = orig_wait(ticket)
        toks, nc = pending_toks.pop(ticket.id)
        seen[len(seen)] = (toks, nc, res)
        return res

    engine.prefill_submit, engine.prefill_wait = gated_submit, recording_wait
    srv = Server([engine], Policy.srjf_calibrated(lam=0.0), lookahead=lookahead)
    try:
        tr = trace()
        futs = [srv.submit(r, YES_NO) for r in tr.requests]
        time.sleep(0.3)
        gate.set()
        results = [f.result(timeout=120) for f in futs]
    finally:
        srv.close()
        del engine.prefill_submit, engine.prefill_wait
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


@pytest.mark.parametrize("lookahead", [False, True])
def test_server_replay_on_gpu_in_real_time(engine, lookahead):
    srv = Server([engine], Policy.srjf_calibrated(), lookahead=lookahead)
    try:
        rep = replay(srv, wl.poisson_arrivals(trace(), 200.0, seed=2), YES_NO)
    finally:
        srv.close()
    assert rep.served == 50 and rep.cache_hit_requests >= 40
    assert rep.p99_latency > 0 and all(r.completion >= r.start >= r.arrival for r in rep.records)


def test_submit_wait_back_to_back_hits_with_distinct_slot_tables(engine):
    """Two prefix hits enqueued before either completes (staging ring): each reads its own pool slots."""
    cfg = llama_ref.Cfg.from_model(TINY)
    w = llama_ref.make_weights(cfg, 42)
    rng = np.random.default_rng([5, 0, 0])
    a = rng.integers(0, 2 ** 32, size=1200, dtype=np.uint32)
    b = rng.integers(0, 2 ** 32, size=1200, dtype=np.uint32)
    sa, sb = list(range(1000, 1075)), list(range(1500, 1575))
    engine.prefill(a, YES_NO, 0, sa)
    engine.prefill(b, YES_NO, 0, sb)
    ta = engine.prefill_submit(a, YES_NO, 1184, sa)
    tb = engine.prefill_submit(b, YES_NO, 1184, sb)
    tc = engine.prefill_submit(a[:640], YES_NO, 0, [])
    rb, ra, rc = engine.prefill_wait(tb), engine.prefill_wait(ta), engine.prefill_wait(tc)
    for toks, res in ((a, ra), (b, rb), (a[:640], rc)):
        logits, _, am = llama_ref.llama_forward(cfg, w, toks, YES_NO)
        assert np.abs(res.logits - logits).max() <= 1e-2 + 5e-3 * np.abs(logits).max()
        assert res.index == am
    assert ra.n_cached == rb.n_cached == 1184 and ra.service_s > 0
    with pytest.raises(Exception):
        engine.prefill_wait(ta)  # consumed

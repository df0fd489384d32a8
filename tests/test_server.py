"""Wall-clock Server (paper_2505_07203_b200/serving.Server) on CPU with a stand-in engine.

The stand-in sleeps for the reference cost model's service time and records the pool ids it receives, so
the worker loop, two-phase admission, scheduling and futures are exercised without a GPU. Every scheduling
decision is checked against the oracle's schedule_next on the same queue snapshot (lock-step shadow).
"""

import threading
import time

import numpy as np

from oracle import sched_ref
from paper_2505_07203_b200 import workload as wl
from paper_2505_07203_b200.engine import PrefillResult
from paper_2505_07203_b200.scheduling import Policy
from paper_2505_07203_b200.serving import Server, replay


class FakeEngine:
    block_tokens = 16

    def __init__(self, pool_blocks=4096, scale=2e-7):
        self.pool_blocks = pool_blocks
        self.capacity_tokens = pool_blocks * 16
        self.scale = scale
        self.calls = []
        self.lock = threading.Lock()

    def prefill(self, tokens, allowed, n_cached=0, pool_block_ids=None):
        n = len(tokens)
        svc = 2e-3 + self.scale * (n - n_cached)
        time.sleep(svc)
        ids = list(pool_block_ids or [])
        assert all(0 <= s < self.pool_blocks for s in ids[: n_cached // 16])
        with self.lock:
            self.calls.append((n, n_cached, ids))
        return PrefillResult(token=allowed[0], index=0, probs=np.array([1.0, 0.0]), logits=np.zeros(2),
                             n_cached=n_cached, service_s=svc)


def small_trace():
    spec = wl.PostRecSpec(users=4, requests_per_user=6, profile_mean=1600, profile_std=200, profile_min=1200,
                          profile_max=2000, suffix_tokens=64)
    return wl.gen_post_recommendation(3, spec)


def test_server_serves_all_and_reuses_prefixes():
    engines = [FakeEngine(), FakeEngine()]
    srv = Server(engines, Policy.srjf_calibrated())
    try:
        rep = replay(srv, wl.poisson_arrivals(small_trace(), 400.0, seed=1), [9642, 2822])
    finally:
        srv.close()
    assert rep.served == 24
    # 4 users x 6 requests: every user's later requests hit its cached profile
    assert rep.cache_hit_requests >= 16
    assert {r.instance for r in rep.records} == {0, 1}
    for e in engines:
        for n, nc, ids in e.calls:
            assert nc % 16 == 0 and len(ids) == n // 16


def test_scheduling_decisions_match_oracle_shadow():
    """Queue everything while the worker is blocked, then compare the order against the oracle."""
    eng = FakeEngine(scale=0.0)
    gate = threading.Event()
    orig = eng.prefill

    def gated(*a, **k):
        gate.wait()
        return orig(*a, **k)

    eng.prefill = gated
    srv = Server([eng], Policy.srjf_calibrated(lam=0.0))
    try:
        trace = small_trace()
        futs = [srv.submit(r, [1, 2]) for r in trace.requests]
        time.sleep(0.2)
        gate.set()
        for f in futs:
            f.result(timeout=30)
    finally:
        srv.close()
    order = [r.id for r in sorted(srv.records, key=lambda r: r.start)]
    # shadow: the oracle picks from the same queue with the same cache evolution (first pick was made before
    # the rest arrived, so replay it the same way)
    cache = sched_ref.PrefixCache(eng.capacity_tokens)
    pending = [dict(id=r.id, n_input=r.n_input, arrival=0.0, frozen_jct=0.0, chain=r.digest_chain(16, {}))
               for r in trace.requests]
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


class AsyncFakeEngine(FakeEngine):
    """Stand-in with the engine's asynchronous API: forwards run back to back on a virtual device timeline."""

    def __init__(self, **kw):
        super().__init__(**kw)
        self.free_at = 0.0
        self.max_inflight = 0
        self.inflight = 0

    def prefill_submit(self, tokens, allowed, n_cached=0, pool_block_ids=None):
        n = len(tokens)
        svc = 2e-3 + self.scale * (n - n_cached)
        now = time.perf_counter()
        self.free_at = max(now, self.free_at) + svc
        with self.lock:
            self.calls.append((n, n_cached, list(pool_block_ids or [])))
            self.inflight += 1
            self.max_inflight = max(self.max_inflight, self.inflight)
        return (self.free_at, svc, allowed[0], n_cached)

    def prefill_done(self, t):
        return time.perf_counter() >= t[0]

    def prefill_wait(self, t):
        d = t[0] - time.perf_counter()
        if d > 0:
            time.sleep(d)
        with self.lock:
            self.inflight -= 1
        return PrefillResult(token=t[2], index=0, probs=np.array([1.0, 0.0]), logits=np.zeros(2), n_cached=t[3],
                             service_s=t[1])


def test_lookahead_keeps_two_forwards_in_flight_and_reuses_prefixes():
    eng = AsyncFakeEngine()
    srv = Server([eng], Policy.srjf_calibrated())
    assert srv.workers[0].lookahead
    try:
        rep = replay(srv, wl.poisson_arrivals(small_trace(), 2000.0, seed=1), [9642, 2822])
    finally:
        srv.close()
    assert rep.served == 24 and rep.cache_hit_requests >= 16
    assert eng.max_inflight == 2  # decided and enqueued while its predecessor ran
    recs = sorted(rep.records, key=lambda r: r.start)
    # back to back on the engine: no record starts before its predecessor completed
    assert all(b.start >= a.completion - 1e-9 for a, b in zip(recs, recs[1:]))
    for n, nc, ids in eng.calls:
        assert nc % 16 == 0 and len(ids) == n // 16


def test_lookahead_decisions_match_oracle_when_all_queued():
    """Everything queued behind a blocked first submit: lookahead takes the same decisions as the oracle."""
    eng = AsyncFakeEngine(scale=0.0)
    gate = threading.Event()
    orig = eng.prefill_submit

    def gated(*a, **k):
        gate.wait()
        return orig(*a, **k)

    eng.prefill_submit = gated
    srv = Server([eng], Policy.srjf_calibrated(lam=0.0))
    try:
        trace = small_trace()
        futs = [srv.submit(r, [1, 2]) for r in trace.requests]
        time.sleep(0.2)
        gate.set()
        for f in futs:
            f.result(timeout=30)
    finally:
        srv.close()
    order = [r.id for r in sorted(srv.records, key=lambda r: (r.start, r.completion))]
    cache = sched_ref.PrefixCache(eng.capacity_tokens)
    pending = [dict(id=r.id, n_input=r.n_input, arrival=0.0, frozen_jct=0.0, chain=r.digest_chain(16, {}))
               for r in trace.requests]
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


def test_least_work_routing_serves_all_and_drains_the_estimates():
    # the optional JCT-aware dispatcher in the wall-clock server: every request served, users sticky,
    # and the outstanding-work counters back to zero once every future has resolved
    from paper_2505_07203_b200.serving import ROUTE_LEAST_WORK

    engines = [FakeEngine(), FakeEngine()]
    srv = Server(engines, Policy.srjf_calibrated(), routing=ROUTE_LEAST_WORK)
    try:
        rep = replay(srv, wl.poisson_arrivals(small_trace(), 400.0, seed=1), [9642, 2822])
    finally:
        srv.close()
    assert rep.served == 24
    by_user = {}
    for r in rep.records:
        by_user.setdefault(r.user_id, set()).add(r.instance)
    assert all(len(v) == 1 for v in by_user.values())
    assert all(abs(x) < 1e-6 for x in srv.router.outstanding)

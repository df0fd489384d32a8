"""Serving loop: router, per-GPU instances (queue + prefix pool + one request in flight), metrics.

Contract of the reference engine loop (ps/sim.py:52-287), which a real engine must honour:
  * Router: sticky user -> instance, first-seen round robin (ps/sim.py:52-66);
  * one request in service per instance; n_cached probed when the request starts; its KV enters the
    instance's prefix cache at completion; events at one timestamp run COMPLETE < FREE < ARRIVE (Q6);
  * latency = completion - arrival, p99 by nearest rank (ps/sim.py:146-151, Q14).

Two drivers share that logic:
  simulate(...)  virtual clock; service time from a callable: the measured GPU forward of a live Engine
                 (trace-driven, every request really runs) or a latency model (e.g. a JctProfile fitted on
                 measured latencies). With the reference's analytic service time it reproduces sim.run
                 record for record (tests/test_serving_parity.py).
  Server         wall clock; one worker thread per engine, submit() -> Future[PrefillResult].
"""

from __future__ import annotations

import heapq
import math
import threading
import time
from concurrent.futures import Future
from dataclasses import dataclass, field
from typing import Callable, Sequence

from .cache import CacheConfig, PrefixCache, block_chain
from .jct import JctProfile
from .scheduling import (POLICY_SRJF, POLICY_SRJF_CALIBRATED, SCORING_PROFILE, Policy, SchedulingError,
                         WaitingRequest, estimate_jct, schedule_next)

EV_COMPLETE, EV_FREE, EV_ARRIVE = 0, 1, 2


class ServingError(ValueError):
    """Invalid serving configuration or trace."""


ROUTE_ROUND_ROBIN = "round_robin"
ROUTE_LEAST_WORK = "least_work"


@dataclass
class Router:
    """Sticky user -> instance assignment (ps/sim.py:52-66).

    round_robin (default, the reference's parity mode): a first-seen user goes to the next instance in turn.
    least_work (optional): a first-seen user goes to the instance with the least outstanding estimated
    work (cache-miss tokens of its queued and running requests; ties to the lowest index), so a few heavy users do
    not pile onto one GPU while another idles; later requests of the user stay there (its prefix is cached there).
    The caller keeps `outstanding` up to date through add_work / done_work."""

    num_instances: int
    assignments: dict = field(default_factory=dict)
    next_rr: int = 0
    mode: str = ROUTE_ROUND_ROBIN
    outstanding: list = field(default_factory=list)

    def __post_init__(self):
        if self.mode not in (ROUTE_ROUND_ROBIN, ROUTE_LEAST_WORK):
            raise ServingError(f"unknown routing mode {self.mode!r}")
        if not self.outstanding:
            self.outstanding = [0.0] * self.num_instances

    def route(self, request) -> int:
        inst = self.assignments.get(request.user_id)
        if inst is None:
            if self.mode == ROUTE_LEAST_WORK:
                inst = min(range(self.num_instances), key=lambda i: (self.outstanding[i], i))
            else:
                inst = self.next_rr % self.num_instances
                self.next_rr += 1
            self.assignments[request.user_id] = inst
        return inst

    def add_work(self, inst: int, work: float):
        self.outstanding[inst] += work

    def done_work(self, inst: int, work: float):
        self.outstanding[inst] -= work


@dataclass(frozen=True)
class RequestRecord:
    id: int
    user_id: int
    instance: int
    arrival: float
    start: float
    completion: float
    n_input: int
    n_cached: int
    token: int = -1  # allowed-token choice (real engine only)

    @property
    def latency(self) -> float:
        return self.completion - self.arrival

    @property
    def service(self) -> float:
        return self.completion - self.start


def p99_nearest_rank(latencies) -> float:
    if not latencies:
        return 0.0
    ordered = sorted(latencies)
    return ordered[max(0, math.ceil(0.99 * len(ordered)) - 1)]


@dataclass(frozen=True)
class ServeReport:
    records: tuple
    mean_latency: float
    p99_latency: float
    throughput: float  # requests / s over the makespan
    cache_hit_tokens: int
    cache_hit_requests: int
    per_instance_utilization: tuple
    makespan: float
    prompt_tokens_per_s: float  # all prompt tokens (n) / makespan
    miss_tokens_per_s: float  # computed tokens (n - n_cached) / makespan

    @property
    def served(self) -> int:
        return len(self.records)

    @property
    def utilization(self) -> float:
        u = self.per_instance_utilization
        return sum(u) / len(u) if u else 0.0


def make_report(records: Sequence[RequestRecord], busy: Sequence[float], first_arrival: float) -> ServeReport:
    if not records:
        return ServeReport((), 0.0, 0.0, 0.0, 0, 0, tuple(0.0 for _ in busy), 0.0, 0.0, 0.0)
    lat = [r.latency for r in records]
    makespan = max(r.completion for r in records) - first_arrival
    tp = len(records) / makespan if makespan > 0 else 0.0
    toks = sum(r.n_input for r in records)
    miss = sum(r.n_input - r.n_cached for r in records)
    return ServeReport(
        records=tuple(records), mean_latency=sum(lat) / len(lat), p99_latency=p99_nearest_rank(lat),
        throughput=tp, cache_hit_tokens=sum(r.n_cached for r in records),
        cache_hit_requests=sum(1 for r in records if r.n_cached > 0),
        per_instance_utilization=tuple((b / makespan if makespan > 0 else 0.0) for b in busy), makespan=makespan,
        prompt_tokens_per_s=toks / makespan if makespan > 0 else 0.0,
        miss_tokens_per_s=miss / makespan if makespan > 0 else 0.0)


@dataclass
class Instance:
    cache: PrefixCache
    queue: list = field(default_factory=list)
    busy: bool = False
    busy_time: float = 0.0


# service_fn(instance_index, waiting_request, n_cached, pool_block_ids) -> seconds, or (seconds, token)
ServiceFn = Callable[[int, WaitingRequest, int, list], object]


def simulate(trace, num_instances: int, policy: Policy, capacity_tokens: int, service_fn: ServiceFn,
             block_tokens: int = 16, jct_profile: JctProfile | None = None, max_input: int | None = None,
             routing: str = ROUTE_ROUND_ROBIN) -> ServeReport:
    """Virtual-clock serving run (the reference's event loop with a pluggable service time). routing: the Router mode
    (round_robin reproduces sim.run; least_work is the optional JCT-aware dispatcher)."""
    reqs = trace.requests
    arr = [r.arrival for r in reqs]
    if any(b < a for a, b in zip(arr, arr[1:])):
        raise ServingError("trace arrivals must be nondecreasing")
    if num_instances < 1:
        raise ServingError("num_instances must be >= 1")
    if max_input is not None:
        over = [r.id for r in reqs if r.n_input > max_input]
        if over:
            from .engine import CapacityError
            raise CapacityError(f"{len(over)} request(s) exceed MIL {max_input}: ids {over[:10]}")
    needs_profile = policy.kind in (POLICY_SRJF, POLICY_SRJF_CALIBRATED) and policy.scoring == SCORING_PROFILE
    if needs_profile and jct_profile is None:
        raise SchedulingError("profile scoring requires a JctProfile")
    if not reqs:
        return make_report([], [0.0] * num_instances, 0.0)

    insts = [Instance(PrefixCache(CacheConfig(capacity_tokens, block_tokens))) for _ in range(num_instances)]
    router = Router(num_instances, mode=routing)
    work: dict = {}  # request id -> (instance, miss-token estimate) while queued or running (least_work routing)
    memo: dict = {}
    events: list = []
    seq = 0
    for r in reqs:
        heapq.heappush(events, (r.arrival, EV_ARRIVE, seq, r))
        seq += 1
    records: list = []

    def start_next(idx: int, now: float):
        nonlocal seq
        inst = insts[idx]
        wr = schedule_next(inst.queue, inst.cache, jct_profile, policy, now)
        inst.queue.remove(wr)
        n_cached = inst.cache.match_chain(wr.chain)
        ncb = n_cached // block_tokens
        slots = inst.cache.slots(wr.chain, ncb)
        adm = inst.cache.begin_insert(wr.chain, now)
        out = service_fn(idx, wr, n_cached, adm.pool_block_ids(ncb, slots))
        service, token = (out if isinstance(out, tuple) else (out, -1))
        inst.busy = True
        inst.busy_time += service
        heapq.heappush(events, (now + service, EV_FREE, seq, idx))
        seq += 1
        heapq.heappush(events, (now + service, EV_COMPLETE, seq, (idx, wr, n_cached, now, adm, token)))
        seq += 1

    while events:
        now, kind, _, payload = heapq.heappop(events)
        if kind == EV_ARRIVE:
            r = payload
            idx = router.route(r)
            inst = insts[idx]
            wr = WaitingRequest(request=r, arrival=now, chain=r.digest_chain(block_tokens, memo))
            if routing == ROUTE_LEAST_WORK:
                est = float(r.n_input - inst.cache.match_chain(wr.chain, committed=True))
                work[r.id] = (idx, est)
                router.add_work(idx, est)
            if policy.kind == POLICY_SRJF:
                wr.frozen_jct = estimate_jct(r.n_input, inst.cache.match_chain(wr.chain, committed=True),
                                             policy.scoring, jct_profile)
            inst.queue.append(wr)
            if not inst.busy:
                start_next(idx, now)
        elif kind == EV_FREE:
            inst = insts[payload]
            inst.busy = False
            if inst.queue:
                start_next(payload, now)
        else:
            idx, wr, n_cached, started, adm, token = payload
            insts[idx].cache.commit(adm, now)
            if routing == ROUTE_LEAST_WORK:
                router.done_work(*work.pop(wr.request.id))
            records.append(RequestRecord(wr.request.id, wr.request.user_id, idx, wr.arrival, started, now,
                                         wr.request.n_input, n_cached, token))
    assert len(records) == len(reqs), "conservation violated"
    return make_report(records, [i.busy_time for i in insts], min(arr))


def engine_service_fn(engines: Sequence, allowed: Sequence[int]) -> ServiceFn:
    """Service function running the real forward on engines[instance]; returns (device seconds, token)."""

    def fn(idx: int, wr: WaitingRequest, n_cached: int, pool_block_ids: list):
        res = engines[idx].prefill(wr.request.tokens, allowed, n_cached, pool_block_ids)
        return res.service_s, res.token

    return fn


class MeasuredServiceFn:
    """Service function that runs each distinct (n_input, n_cached) request shape once on a live Engine and
    reuses the measured device seconds (every shape in the trace is a real forward on the GPU).

    TIMING ONLY. All instances share one engine's measurements (request-level DP replicas on identical GPUs). A
    reused measurement runs no forward, so the blocks the loop's cache admitted for that request hold no K/V in the
    engine's pool, and instances simulated on one engine would name colliding pool slots: the returned token of a
    reused shape is None, and no pool content produced under this function may be trusted.
    """

    def __init__(self, engine, allowed: Sequence[int]):
        self.engine = engine
        self.allowed = list(allowed)
        self.memo: dict = {}
        self.forwards = 0

    def __call__(self, idx: int, wr: WaitingRequest, n_cached: int, pool_block_ids: list):
        key = (wr.request.n_input, n_cached)
        hit = self.memo.get(key)
        if hit is None:
            res = self.engine.prefill(wr.request.tokens, self.allowed, n_cached, pool_block_ids)
            self.memo[key] = (res.service_s, None)
            self.forwards += 1
            return res.service_s, res.token
        return hit


class ReplayServiceFn:
    """Service function that runs every request for real, in the order the serving loop executes them, and
    records each request's device seconds; a later run that meets the same (request, n_cached) reuses them.

    Run once over the saturation trace (every request at t = 0, so the loop's own order), this measures each
    request in the GPU state the serving order puts it in: a prefix hit right after a cold 20k forward runs at the
    clocks the power cap left (tools/hit_after_cold.py), later hits of the session at recovered clocks. Shapes a
    later run meets that the replay did not (a different cache state) fall back to one measured forward per shape.

    TIMING ONLY once `recording` is off: reused entries run no forward (their admitted pool slots get no K/V) and
    return token None. Under world > 1 every simulated instance drives this one engine, so their pool slot numbers
    collide; bench.py's multi-GPU path gives each rank its own engine and shard of the trace instead.
    """

    def __init__(self, engine, allowed: Sequence[int]):
        self.engine = engine
        self.allowed = list(allowed)
        self.by_request: dict = {}
        self.by_shape: dict = {}
        self.forwards = 0
        self.recording = True  # the first (saturation) run records per request; set False afterwards

    def __call__(self, idx: int, wr: WaitingRequest, n_cached: int, pool_block_ids: list):
        key = (wr.request.id, n_cached)
        hit = self.by_request.get(key)
        if hit is None:
            shape = (wr.request.n_input, n_cached)
            if self.recording or shape not in self.by_shape:
                res = self.engine.prefill(wr.request.tokens, self.allowed, n_cached, pool_block_ids)
                self.forwards += 1
                hit = (res.service_s, res.token)
                self.by_shape.setdefault(shape, hit)
            else:
                hit = (self.by_shape[shape][0], None)
            if self.recording:
                self.by_request[key] = hit
            return hit
        return hit[0], None


def shard_trace(trace, rank: int, world: int):
    """Requests the sticky router sends to instance `rank` (request-level DP: each GPU serves its own users).

    Routing depends only on first-arrival order of users, so every rank computes the same assignment locally;
    no collective is needed on the data path.
    """
    router = Router(world)
    mine = tuple(r for r in trace.requests if router.route(r) == rank)
    return type(trace)(trace.name, trace.seed, mine)


def merge_records(per_rank: Sequence[Sequence[RequestRecord]], world: int) -> ServeReport:
    """Global report from per-rank records (rank r's records carry instance 0 locally -> r)."""
    recs, busy = [], []
    for rank, rr in enumerate(per_rank):
        b = 0.0
        for r in rr:
            recs.append(RequestRecord(r.id, r.user_id, rank, r.arrival, r.start, r.completion, r.n_input,
                                      r.n_cached, r.token))
            b += r.service
        busy.append(b)
    recs.sort(key=lambda r: (r.completion, r.id))
    first = min((r.arrival for r in recs), default=0.0)
    return make_report(recs, busy, first)


def sweep_rates(trace, rates: Sequence[float], seed: int, run: Callable, keep_sessions: bool = True):
    """Run `run(arrived_trace)` at each Poisson rate; returns [(rate, ServeReport)]."""
    from .workload import poisson_arrivals

    return [(q, run(poisson_arrivals(trace, q, seed=seed, keep_sessions=keep_sessions))) for q in rates]


def qps_at_slo(results, slo_s: float) -> float:
    """Largest swept rate whose p99 latency meets the SLO (0 if none)."""
    ok = [q for q, rep in results if rep.p99_latency <= slo_s]
    return max(ok) if ok else 0.0


def refine_qps(results, slo_s: float, evaluate: Callable, steps: int = 5):
    """Bisect between the largest swept rate that meets the SLO and the next swept rate above it that misses, so
    QPS@SLO is resolved to (gap / 2^steps) instead of the sweep's grid. evaluate(rate) -> ServeReport. Returns the
    results with the bisection points added, sorted by rate."""
    res = sorted(results, key=lambda x: x[0])
    ok = [q for q, rep in res if rep.p99_latency <= slo_s]
    if not ok:
        return res
    lo = max(ok)
    above = [q for q, rep in res if q > lo and rep.p99_latency > slo_s]
    if not above:
        return res
    hi = min(above)
    for _ in range(steps):
        mid = 0.5 * (lo + hi)
        rep = evaluate(mid)
        res.append((mid, rep))
        if rep.p99_latency <= slo_s:
            lo = mid
        else:
            hi = mid
    return sorted(res, key=lambda x: x[0])


# ------------------------------------------------------------------ wall-clock server


@dataclass
class _Job:
    wr: WaitingRequest
    allowed: tuple
    future: Future


class _Worker(threading.Thread):
    """One engine's serving loop.

    lookahead=False: decide, run, commit, repeat -- every decision is taken when the engine frees up, the
    reference's event order (ps/sim.py:211-229), and the host-side work (schedule_next, cache probes, slot tables,
    enqueueing the forward) sits between forwards with the GPU idle.
    lookahead=True (default, engines with prefill_submit): up to two forwards in flight on the engine stream. As soon
    as a forward is enqueued the loop takes the next decision (schedule_next, begin_insert, commit) and enqueues it
    behind, so the host work of request i+1 overlaps the forward of request i and the GPU runs back to back. A
    decision is then taken when its predecessor starts rather than when it completes: requests arriving during that
    forward compete from the following decision on. The admission is committed at decision time; the predecessor's
    forward (same stream) completes before this one's starts, so K/V it admits are in the pool when they are read,
    and a slot this decision evicts is overwritten only after the predecessor has read it. One thread per engine:
    the C-ABI calls release the GIL, and no second Python thread competes for it.
    """

    DEPTH = 2  # forwards in flight per engine (the staging ring holds 4)

    def __init__(self, server: "Server", idx: int, engine, lookahead: bool = True):
        super().__init__(daemon=True, name=f"prefillonly-worker-{idx}")
        self.server, self.idx, self.engine = server, idx, engine
        self.inst = Instance(PrefixCache(CacheConfig(engine.capacity_tokens, engine.block_tokens)))
        self.jobs: dict = {}
        self.cv = threading.Condition()
        self.stop = False
        self.lookahead = lookahead and hasattr(engine, "prefill_submit")

    def enqueue(self, job: _Job, now: float):
        with self.cv:
            if self.server.policy.kind == POLICY_SRJF:
                job.wr.frozen_jct = estimate_jct(job.wr.request.n_input,
                                                 self.inst.cache.match_chain(job.wr.chain, committed=True),
                                                 self.server.policy.scoring, self.server.jct_profile)
            self.jobs[id(job.wr)] = job
            self.inst.queue.append(job.wr)
            self.cv.notify()

    def _decide(self, now: float):
        """schedule_next + cache probe + admission (caller holds self.cv)."""
        srv = self.server
        bt = self.engine.block_tokens
        wr = schedule_next(self.inst.queue, self.inst.cache, srv.jct_profile, srv.policy, now)
        self.inst.queue.remove(wr)
        job = self.jobs.pop(id(wr))
        n_cached = self.inst.cache.match_chain(wr.chain)
        ncb = n_cached // bt
        slots = self.inst.cache.slots(wr.chain, ncb)
        adm = self.inst.cache.begin_insert(wr.chain, now)
        return wr, job, n_cached, adm.pool_block_ids(ncb, slots), adm

    def _finish(self, wr, job, n_cached, res, start, done):
        rec = RequestRecord(wr.request.id, wr.request.user_id, self.idx, wr.arrival, start, done,
                            wr.request.n_input, n_cached, res.token)
        self.server._record(rec)
        job.future.set_result(res)

    def run(self):
        if self.lookahead:
            return self._pipelined()
        srv = self.server
        eng = self.engine
        while True:
            with self.cv:
                while not self.inst.queue and not self.stop:
                    self.cv.wait()
                if self.stop and not self.inst.queue:
                    return
                now = srv.clock()
                wr, job, n_cached, ids, adm = self._decide(now)
            try:
                res = eng.prefill(wr.request.tokens, job.allowed, n_cached, ids)
            except Exception as exc:  # the forward failed: its admitted blocks hold no K/V
                with self.cv:
                    self.inst.cache.abort(adm)
                job.future.set_exception(exc)
                continue
            done = srv.clock()
            with self.cv:
                self.inst.cache.commit(adm, done)
                self.inst.busy_time += done - now
            self._finish(wr, job, n_cached, res, now, done)

    def _drop_admission(self, adm):
        """A committed admission whose forward failed: its new blocks never received K/V."""
        cache = self.inst.cache
        for b, _ in reversed(adm.admit):
            d = adm.chain[b]
            if d in cache._blocks and cache._blocks[d].children == 0:
                cache._remove(d)
        cache.version += 1

    def _pipelined(self):
        srv = self.server
        eng = self.engine
        inflight: list = []  # [wr, job, n_cached, adm, ticket, t_submit], oldest first
        last_done = 0.0
        while True:
            plan = None
            with self.cv:
                while not self.stop and not self.inst.queue and not inflight:
                    self.cv.wait()
                if self.stop and not self.inst.queue and not inflight:
                    return
                if self.inst.queue and len(inflight) < self.DEPTH:
                    now = srv.clock()
                    plan = self._decide(now)
                    self.inst.cache.commit(plan[4], now)
            if plan is not None:
                wr, job, n_cached, ids, adm = plan
                try:
                    ticket = eng.prefill_submit(wr.request.tokens, job.allowed, n_cached, ids)
                except Exception as exc:
                    with self.cv:
                        self._drop_admission(adm)
                    job.future.set_exception(exc)
                    continue
                inflight.append([wr, job, n_cached, adm, ticket, now])
                if len(inflight) < self.DEPTH:
                    continue  # keep the engine fed: decide the next one while this forward runs
            wr, job, n_cached, adm, ticket, t_sub = inflight[0]
            if len(inflight) < self.DEPTH and not eng.prefill_done(ticket):
                # one forward in flight and nothing to plan: wake on an arrival or poll the completion
                with self.cv:
                    if not self.inst.queue and not self.stop:
                        self.cv.wait(timeout=2e-4)
                continue
            inflight.pop(0)
            try:
                res = eng.prefill_wait(ticket)
            except Exception as exc:
                with self.cv:
                    self._drop_admission(adm)
                job.future.set_exception(exc)
                continue
            done = srv.clock()
            start = max(t_sub, last_done)  # it ran behind its predecessor on the engine stream
            last_done = done
            with self.cv:
                self.inst.busy_time += done - start
            self._finish(wr, job, n_cached, res, start, done)


class Server:
    """Request-level data parallelism over engines (one per GPU), SRJF-calibrated by default."""

    def __init__(self, engines: Sequence, policy: Policy | None = None, jct_profile: JctProfile | None = None,
                 lookahead: bool = True, routing: str = ROUTE_ROUND_ROBIN):
        if not engines:
            raise ServingError("need at least one engine")
        self.policy = policy or Policy.srjf_calibrated()
        self.jct_profile = jct_profile
        self.router = Router(len(engines), mode=routing)
        self._t0 = time.monotonic()
        self._lock = threading.Lock()
        self.records: list = []
        self._memo: dict = {}
        self.workers = [_Worker(self, i, e, lookahead) for i, e in enumerate(engines)]
        for w in self.workers:
            w.start()

    def clock(self) -> float:
        return time.monotonic() - self._t0

    def reset_clock(self):
        self._t0 = time.monotonic()

    def _record(self, rec: RequestRecord):
        with self._lock:
            self.records.append(rec)

    def submit(self, request, allowed: Sequence[int]) -> Future:
        """Queue one request (duck type .id, .user_id, .n_input, .tokens); resolves to a PrefillResult.

        Thread-safe: routing (first-seen round robin, or least outstanding work) and the digest memo are updated under
        the server lock."""
        with self._lock:
            idx = self.router.route(request)
            bt = self.workers[idx].engine.block_tokens
            chain = request.digest_chain(bt, self._memo) if hasattr(request, "digest_chain") else \
                block_chain(request.tokens, bt)
        wr = WaitingRequest(request=request, arrival=self.clock(), chain=chain)
        fut: Future = Future()
        if self.router.mode == ROUTE_LEAST_WORK:
            w = self.workers[idx]
            with w.cv:  # the worker thread owns the cache
                est = float(request.n_input - w.inst.cache.match_chain(chain, committed=True))
            with self._lock:
                self.router.add_work(idx, est)

            def _done(_f, idx=idx, est=est):
                with self._lock:
                    self.router.done_work(idx, est)

            fut.add_done_callback(_done)
        self.workers[idx].enqueue(_Job(wr, tuple(allowed), fut), wr.arrival)
        return fut

    def report(self) -> ServeReport:
        with self._lock:
            recs = sorted(self.records, key=lambda r: r.completion)
        first = min((r.arrival for r in recs), default=0.0)
        return make_report(recs, [w.inst.busy_time for w in self.workers], first)

    def close(self):
        for w in self.workers:
            with w.cv:
                w.stop = True
                w.cv.notify()
        for w in self.workers:
            w.join()


def replay(server: Server, trace, allowed: Sequence[int]) -> ServeReport:
    """Inject the trace's arrivals in wall-clock time, wait for every completion, report."""
    server.reset_clock()
    futs = []
    for r in trace.requests:
        delay = r.arrival - server.clock()
        if delay > 0:
            time.sleep(delay)
        futs.append(server.submit(r, allowed))
    for f in futs:
        f.result()
    return server.report()

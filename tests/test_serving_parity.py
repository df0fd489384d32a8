"""Serving loop (paper_2505_07203_b200/serving.py) reproduces the reference event loop record for record.

With the reference's analytic service time (execute_time, prefillonly branch, ps/costs.py:275-280) as the
pluggable service function, `simulate` must emit exactly sim.run's records (ps/sim.py:162-287): same
instance routing, start/completion times (float-equal), and n_cached per request.
"""

import numpy as np
import pytest

from golden_util import golden
from paper_2505_07203_b200 import workload as wl
from paper_2505_07203_b200.scheduling import Policy
from paper_2505_07203_b200.serving import Router, p99_nearest_rank, simulate

POL = {"fifo": Policy.fifo(), "srjf": Policy.srjf_static(), "srjf-calibrated": Policy.srjf_calibrated()}


def small_trace(g):
    lens = wl.post_rec_profile_lengths(g["trace_seed"])[: g["users"]]
    reqs = []
    for u, plen in enumerate(lens):
        for _ in range(g["per_user"]):
            reqs.append(wl.Request(len(reqs), u, 0.0, plen // 8, plen // 8 + 150, g["trace_seed"]))
    return wl.Trace("post-rec-small", g["trace_seed"], tuple(reqs))


@pytest.mark.parametrize("k", range(12))
def test_simulate_matches_reference_sim_run(k):
    g = golden()["sim_runs"]
    run = g["runs"][k]
    trace = wl.poisson_arrivals(small_trace(g), run["rate"], seed=g["arrival_seed"], keep_sessions=True)

    def svc(idx, wr, n_cached, ids):
        n = wr.request.n_input
        return g["c_fixed"] + g["c_linear"] * (n - n_cached) + g["c_attn"] * ((n * n - n_cached * n_cached) / 2.0)

    rep = simulate(trace, run["instances"], POL[run["policy"]], g["capacity_tokens"], svc)
    got = [[r.id, r.instance, r.start, r.completion, r.n_cached] for r in rep.records]
    assert got == run["records"]
    assert rep.p99_latency == run["p99"] and rep.mean_latency == pytest.approx(run["mean"], rel=1e-12)
    assert rep.cache_hit_requests == run["hit_requests"] and rep.cache_hit_tokens == run["hit_tokens"]


def test_worked_example_orders_and_hits():
    trace, cap = wl.worked_example()
    exp = golden()["worked_example"]
    for name, pol in POL.items():
        rep = simulate(trace, 1, pol, cap, lambda i, w, nc, ids: 0.02 + 1e-4 * (w.request.n_input - nc))
        order = [r.id for r in sorted(rep.records, key=lambda r: r.start)]
        assert order == exp[name]["order"] and rep.cache_hit_requests == exp[name]["hits"]


def test_router_sticky_round_robin_split():
    class R:
        def __init__(self, u):
            self.user_id = u

    r = Router(8)
    inst = [r.route(R(u)) for u in range(20)]
    assert [r.route(R(u)) for u in range(20)] == inst
    counts = np.bincount(inst, minlength=8).tolist()
    assert counts == [3, 3, 3, 3, 2, 2, 2, 2]


def test_p99_nearest_rank():
    assert p99_nearest_rank([]) == 0.0
    assert p99_nearest_rank(list(range(1, 101))) == 99
    assert p99_nearest_rank([5.0]) == 5.0
    assert p99_nearest_rank(list(range(1, 201))) == 198


def test_service_fn_receives_pool_plan():
    trace, cap = wl.worked_example()
    seen = []

    def svc(idx, w, nc, ids):
        seen.append((w.request.id, nc, list(ids)))
        return 0.1

    simulate(trace, 1, Policy.srjf_calibrated(), cap, svc)
    # the second request (D) reuses A's 64 blocks: its first 64 pool ids are A's admission slots
    (a_id, a_nc, a_ids), (d_id, d_nc, d_ids) = seen[0], seen[1]
    assert (a_id, d_id, a_nc, d_nc) == (0, 3, 0, 1024)
    assert d_ids[:64] == a_ids[:64] and len(d_ids) == 2944 // 16


def test_replay_service_fn_records_each_request_once_and_reuses():
    """ReplayServiceFn: the saturation run executes every request (in serving order) and records it; later runs
    reuse the recorded (request, n_cached) times and measure only unseen shapes."""
    from paper_2505_07203_b200 import workload as wl
    from paper_2505_07203_b200.scheduling import Policy
    from paper_2505_07203_b200.serving import ReplayServiceFn, simulate

    class Eng:
        def __init__(self):
            self.calls = 0

        def prefill(self, tokens, allowed, n_cached=0, pool_block_ids=None):
            self.calls += 1

            class R:
                service_s = 1e-3 * (len(tokens) - n_cached) / 1000 + 1e-4 * self.calls
                token = allowed[0]
            return R()

    trace = wl.gen_post_recommendation(0, wl.POSTREC_20K)
    trace = type(trace)(trace.name, trace.seed, trace.requests[:120])
    eng = Eng()
    svc = ReplayServiceFn(eng, [1, 2])
    rep0 = simulate(wl.zero_arrivals(trace), 1, Policy.srjf_calibrated(), 400_000, svc)
    assert eng.calls == len(trace.requests) == len(svc.by_request)  # every request ran for real, once
    svc.recording = False
    calls = eng.calls
    rep1 = simulate(wl.zero_arrivals(trace), 1, Policy.srjf_calibrated(), 400_000, svc)
    assert eng.calls == calls  # same order and cache state: all reused
    assert rep1.p99_latency == rep0.p99_latency


def test_refine_qps_bisects_to_the_knee():
    from types import SimpleNamespace

    from paper_2505_07203_b200.serving import qps_at_slo, refine_qps

    knee = 7.3
    rep = lambda q: SimpleNamespace(p99_latency=1.0 if q <= knee else 10.0)  # noqa: E731
    grid = [(q, rep(q)) for q in (2.0, 4.0, 6.0, 8.0, 10.0)]
    assert qps_at_slo(grid, 2.0) == 6.0
    calls = []
    out = refine_qps(grid, 2.0, lambda q: calls.append(q) or rep(q), steps=6)
    assert len(calls) == 6 and all(6.0 < q < 8.0 for q in calls)
    best = qps_at_slo(out, 2.0)
    assert knee - 2.0 / 2 ** 6 <= best <= knee
    assert [q for q, _ in out] == sorted(q for q, _ in out)
    # nothing to refine: every rate passes, or none does
    never = lambda q: 1 / 0  # noqa: E731  (must not be called)
    assert [q for q, _ in refine_qps([(1.0, rep(1.0))], 2.0, never)] == [1.0]
    assert [q for q, _ in refine_qps([(9.0, rep(9.0))], 2.0, never)] == [9.0]

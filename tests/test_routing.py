"""The optional JCT-aware dispatcher: Router(mode="least_work") sends a first-seen user to the instance
with the least outstanding cache-miss work. Round robin stays the default and reproduces the reference (the parity
tests in test_serving_parity.py run the default); these tests check the option's behaviour."""

import numpy as np
import pytest

from paper_2505_07203_b200 import workload as wl
from paper_2505_07203_b200.scheduling import Policy
from paper_2505_07203_b200.serving import ROUTE_LEAST_WORK, ROUTE_ROUND_ROBIN, Router, ServingError, simulate
from paper_2505_07203_b200.workload import Request, Trace


class _R:
    def __init__(self, uid):
        self.user_id = uid


def test_round_robin_is_default_and_sticky():
    r = Router(3)
    assert [r.route(_R(u)) for u in (10, 11, 12, 13, 10, 11)] == [0, 1, 2, 0, 0, 1]


def test_least_work_picks_least_loaded_then_sticks():
    r = Router(3, mode=ROUTE_LEAST_WORK)
    assert r.route(_R(1)) == 0  # all idle: lowest index
    r.add_work(0, 20_000)
    assert r.route(_R(2)) == 1
    r.add_work(1, 5_000)
    assert r.route(_R(3)) == 2
    r.add_work(2, 1_000)
    assert r.route(_R(4)) == 2  # least outstanding
    r.done_work(0, 20_000)
    assert r.route(_R(5)) == 0
    assert r.route(_R(1)) == 0 and r.route(_R(2)) == 1  # sticky


def test_unknown_mode_rejected():
    with pytest.raises(ServingError):
        Router(2, mode="random")


def _skewed_trace():
    # 16 users on 8 GPUs; users 0 and 8 send 12 long requests each, the others 2 short ones, all at t = 0 in user
    # order: round robin puts both heavy users on GPU 0 (SURVEY Q13's imbalance), least-work does not
    reqs, rid = [], 0
    for u in range(16):
        heavy = u % 8 == 0
        for _ in range(12 if heavy else 2):
            n = 20_000 if heavy else 4_000
            reqs.append(Request(rid, u, 0.0, n // 2, n, 0))
            rid += 1
    return Trace("skewed", 0, tuple(reqs))


def _svc(idx, wr, n_cached, pool_block_ids):
    return 1e-5 * (wr.request.n_input - n_cached) + 1e-3


def test_least_work_balances_a_skewed_trace():
    tr = _skewed_trace()
    rr = simulate(tr, 8, Policy.fifo(), 10_000_000, _svc)
    lw = simulate(tr, 8, Policy.fifo(), 10_000_000, _svc, routing=ROUTE_LEAST_WORK)
    assert len(rr.records) == len(lw.records) == len(tr.requests)
    # round robin stacks both heavy users on GPU 0; least-work spreads them: shorter makespan and tail
    assert {r.instance for r in rr.records if r.user_id in (0, 8)} == {0}
    assert len({r.instance for r in lw.records if r.user_id in (0, 8)}) == 2
    assert lw.makespan < 0.6 * rr.makespan
    assert lw.p99_latency < rr.p99_latency


def test_round_robin_routing_argument_matches_default():
    tr = wl.poisson_arrivals(_skewed_trace(), 20.0, seed=1, keep_sessions=True)
    a = simulate(tr, 4, Policy.srjf_calibrated(), 1_000_000, _svc)
    b = simulate(tr, 4, Policy.srjf_calibrated(), 1_000_000, _svc, routing=ROUTE_ROUND_ROBIN)
    assert [(r.id, r.instance, r.start, r.completion) for r in a.records] == \
        [(r.id, r.instance, r.start, r.completion) for r in b.records]

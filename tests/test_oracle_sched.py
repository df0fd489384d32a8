"""oracle/sched_ref.py pinned against fixtures generated from the reference (tests/golden/make_golden.py)."""

import numpy as np
import pytest

from golden_util import golden
from oracle import sched_ref


def test_block_chains():
    for c in golden()["block_chains"]:
        toks = np.random.default_rng([c["seed"], 77]).integers(0, 2 ** 32, size=c["n"], dtype=np.uint32)
        assert [d.hex() for d in sched_ref.block_chain(toks, c["bt"])] == c["chain"]


def test_cache_op_sequence():
    g = golden()["cache_ops"]
    chains = [sched_ref.block_chain(np.array(s, dtype=np.uint32), g["bt"]) for s in g["seqs"]]
    cache = sched_ref.PrefixCache(g["capacity_tokens"], g["bt"])
    for op in g["ops"]:
        if op["op"] == "insert":
            assert cache.insert_chain(chains[op["seq"]], op["now"]) == op["out"]
        elif op["op"] == "match":
            assert cache.match_chain(chains[op["seq"]]) == op["out"]
        else:
            try:
                out = cache.evict_to(op["need"], protect=chains[op["seq"]])
            except ValueError:
                out = None
            if op["out"] >= 0:
                assert out == op["out"]
            else:
                assert out is None
        assert cache.used_tokens == op["used"]
    assert sorted(d.hex() for d in cache.blocks) == g["final_resident"]


def test_scheduler_orders():
    g = golden()["scheduler"]
    for case in g["cases"]:
        now = case["now"]
        for name, order in case["orders"].items():
            pol = {"fifo": ("fifo", 0.5, "proxy"), "srjf": ("srjf", 0.5, "proxy"), "cal0": ("cal", 0.0, "proxy"),
                   "cal05": ("cal", 0.5, "proxy"), "cal500": ("cal", 500.0, "proxy"),
                   "calprof": ("cal", 0.01, "profile")}[name]

            class Probe:  # cache stand-in answering the recorded probes
                def __init__(self, q):
                    self.q = {w["id"]: w["n_cached"] for w in q}

                def match_chain(self, chain):
                    return self.q[chain]

            pending = [dict(w, chain=w["id"]) for w in case["queue"]]
            got = []
            while pending:
                w = sched_ref.schedule_next(pending, Probe(case["queue"]), pol[0], now, pol[1], pol[2],
                                            (2e-5, -1.5e-5, 0.01))
                got.append(w["id"])
                pending.remove(w)
            assert got == order, (name, got, order)


def sim_trace(g):
    from paper_2505_07203_b200 import workload as wl  # the generator is validated separately

    spec_len = wl.post_rec_profile_lengths(g["trace_seed"])[: g["users"]]
    reqs = []
    for u, plen in enumerate(spec_len):
        plen = plen // 8
        for _ in range(g["per_user"]):
            reqs.append(wl.Request(len(reqs), u, 0.0, plen, plen + 150, g["trace_seed"]))
    return wl.Trace("post-rec-small", g["trace_seed"], tuple(reqs))


@pytest.mark.parametrize("k", range(12))
def test_event_loop_records(k):
    from paper_2505_07203_b200 import workload as wl

    g = golden()["sim_runs"]
    run = g["runs"][k]
    trace = wl.poisson_arrivals(sim_trace(g), run["rate"], seed=g["arrival_seed"], keep_sessions=True)
    memo = {}
    reqs = [{"id": r.id, "user_id": r.user_id, "arrival": r.arrival, "n_input": r.n_input,
             "chain": r.digest_chain(16, memo)} for r in trace.requests]

    def svc(n, nc):  # execute_time, prefillonly branch (ps/costs.py:275-280)
        return g["c_fixed"] + g["c_linear"] * (n - nc) + g["c_attn"] * ((n * n - nc * nc) / 2.0)

    pol = {"fifo": "fifo", "srjf": "srjf", "srjf-calibrated": "cal"}[run["policy"]]
    recs = sched_ref.run(reqs, run["instances"], pol, g["capacity_tokens"], svc)
    assert [list(r) for r in recs] == run["records"]

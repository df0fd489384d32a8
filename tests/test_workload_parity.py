"""Product workload generators reproduce the reference traces (ps/workload.py) from the same seeds."""

import hashlib

import numpy as np

from golden_util import golden
from paper_2505_07203_b200 import workload as wl


def test_lengths_tokens_and_chain():
    g = golden()["workload"]
    assert wl.post_rec_profile_lengths(0) == g["post_rec_profile_lengths"]
    assert wl.credit_lengths(0) == g["credit_lengths"]
    r = wl.gen_post_recommendation(0).requests[51]
    assert r.tokens[:8].tolist() == g["post_rec_tokens_req51_head"]
    assert r.suffix_tokens[:4].tolist() == g["post_rec_tokens_req51_suffix"]
    assert r.suffix_tokens[0] == 51
    assert hashlib.sha256(b"".join(r.digest_chain(16, {}))).hexdigest() == g["post_rec_req51_chain_sha256"]


def test_poisson_arrivals():
    g = golden()["workload"]
    a = wl.poisson_arrivals(wl.gen_post_recommendation(0), 2.5, seed=1, keep_sessions=True)
    assert [[r.id, r.arrival] for r in a.requests[:60]] == g["poisson_keep"]
    b = wl.poisson_arrivals(wl.gen_credit_verification(0), 0.7, seed=2, keep_sessions=False)
    assert [[r.id, r.arrival] for r in b.requests] == g["poisson_interleave"]


def test_baseline_shapes_and_trace_io(tmp_path):
    t = wl.gen_post_recommendation(0, wl.POSTREC_20K)
    assert len(t) == 40 * 50 and 16_850 + 150 <= min(r.n_input for r in t.requests)
    assert max(r.n_input for r in t.requests) <= 22_850 + 150
    c = wl.gen_credit_verification(0, wl.CREDIT_10K_60K)
    assert all(10_000 <= r.n_input <= 60_000 for r in c.requests)
    p = tmp_path / "t.csv"
    wl.save_trace(wl.poisson_arrivals(t, 3.0, seed=0), p)
    back = wl.load_trace(p)
    assert [r.arrival for r in back.requests] == [r.arrival for r in wl.poisson_arrivals(t, 3.0, seed=0).requests]

"""JCT estimator (paper_2505_07203_b200/jct.py): the reference's fit anchors (pkg/tests/test_jct.py)."""

import numpy as np
import pytest

from golden_util import golden
from paper_2505_07203_b200 import jct


def test_grid_fit_matches_reference():
    g = golden()["geometry_jct"]
    sr = golden()["sim_runs"]

    def svc(n, nc):  # execute_time prefillonly branch with the l4/llama-8b CostParams
        return sr["c_fixed"] + sr["c_linear"] * (n - nc) + sr["c_attn"] * ((n * n - nc * nc) / 2.0)

    prof = jct.fit(jct.generate_samples(svc, max_input=min(g["l4_hybrid_mil"], 60_000)))
    assert prof.fit_r2 == pytest.approx(0.963387, abs=5e-7)
    assert np.allclose([prof.coef_input, prof.coef_cached, prof.intercept, prof.fit_r2], g["grid_fit"], rtol=1e-9)


def test_exact_recovery_and_errors(tmp_path):
    s = [jct.JctSample(n, nc, 1e-4 * n - 5e-5 * nc + 0.02) for n, nc in jct.profile_grid(5000)]
    p = jct.fit(s)
    assert p.coef_input == pytest.approx(1e-4) and p.coef_cached == pytest.approx(-5e-5)
    assert p.intercept == pytest.approx(0.02) and p.fit_r2 == pytest.approx(1.0)
    with pytest.raises(jct.FitError):
        jct.fit(s[:2])
    with pytest.raises(jct.FitError):
        jct.fit([jct.JctSample(1000, nc, 1.0) for nc in (0, 100, 200)])
    assert jct.proxy_miss(14000, 11000) == golden()["geometry_jct"]["proxy_miss_14000_11000"] == 3000
    assert jct.get_jct(jct.JctProfile(1e-5, 0, 0.1, 1), 1000, 500) == pytest.approx(0.11)
    f = tmp_path / "p.txt"
    jct.save_profile(p, f)
    assert jct.load_profile(f) == p
    assert jct.pearson([1, 2, 3], [2, 4, 6.5]) > 0.99

"""KV-manager sizing (paper_2505_07203_b200/geometry.py) against the reference's anchors
(pkg/tests/test_geometry.py) and the hybrid-prefill MIL claim on a 180 GB B200."""

import pytest

from golden_util import golden
from paper_2505_07203_b200 import geometry as G
from paper_2505_07203_b200.config import LLAMA_3_1_8B, QWEN_2_5_32B, TINY


def test_kv_bytes_and_spike_match_reference():
    assert list(G.kv_bytes_per_token(LLAMA_3_1_8B)) == golden()["geometry_jct"]["kv_bytes_per_token"]
    assert G.kv_bytes_per_token(LLAMA_3_1_8B) == (4096, 131072)
    assert G.intermediate_bytes_per_token(LLAMA_3_1_8B) == 57_344  # 28,672 bf16 scalars
    assert LLAMA_3_1_8B.weight_bytes == 16_060_522_496  # llama-3.1-8b.preset weight_bytes (8,030,261,248 params)


def test_flop_formulas_match_reference():
    g = golden()["geometry_jct"]
    assert LLAMA_3_1_8B.linear_flops_per_token() == g["linear_flops_per_token"]
    assert LLAMA_3_1_8B.attn_flops_per_pair() == g["attn_flops_per_pair"]


def test_hybrid_mil_on_b200_exceeds_128k():
    mil = G.max_input_length(LLAMA_3_1_8B, mode=G.HYBRID)
    assert mil > 131_072 * 10  # one-layer KV + chunked MLP: millions of tokens fit beside 16 GB of weights
    full = G.max_input_length(LLAMA_3_1_8B, mode=G.FULL)
    assert 131_072 < full < mil
    assert G.max_input_length(QWEN_2_5_32B, mode=G.HYBRID) > 60_000


def test_peak_ordering_and_ratio():
    n = 20_000
    peaks = {m: G.peak_prefill_memory(LLAMA_3_1_8B, n, m) for m in (G.FULL, G.KV_DISCARD, G.CHUNKED, G.HYBRID)}
    assert peaks[G.HYBRID] < peaks[G.CHUNKED] < peaks[G.FULL]
    assert peaks[G.HYBRID] < peaks[G.KV_DISCARD] < peaks[G.FULL]
    assert 0 < G.peak_ratio(LLAMA_3_1_8B, 131_072) < 0.6


def test_prefix_capacity_and_errors():
    cap = G.prefix_cache_capacity(LLAMA_3_1_8B, 20_000)
    assert 1_000_000 < cap < 1_400_000  # ~140 GB of 128 KiB/token prefix K/V
    with pytest.raises(G.GeometryError):
        G.prefix_cache_capacity(LLAMA_3_1_8B, 10 ** 9)
    with pytest.raises(G.GeometryError):
        G.peak_prefill_memory(TINY, 0)
    assert G.largest_fitting(lambda n: n, 10) == 10

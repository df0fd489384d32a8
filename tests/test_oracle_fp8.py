"""The oracle's E4M3 rounding and per-row quantisation (oracle/llama_ref.py), pinned against torch's own
float8_e4m3fn conversion on CPU; and the FP8 presets' byte accounting."""

import numpy as np
import pytest

from oracle import llama_ref
from paper_2505_07203_b200 import geometry
from paper_2505_07203_b200.config import LLAMA_3_3_70B_FP8, QWEN_2_5_32B, QWEN_2_5_32B_FP8, TINY_FP8

torch = pytest.importorskip("torch")


def test_e4m3_round_matches_torch_on_every_code_and_midpoint():
    codes = torch.arange(256, dtype=torch.uint8).view(torch.float8_e4m3fn).float().numpy().astype(np.float64)
    finite = np.unique(codes[np.isfinite(codes)])
    assert finite.max() == 448.0 and len(finite) == 253  # +-0 collapse; 0x7F / 0xFF are NaN
    assert np.array_equal(llama_ref.e4m3_round(finite), finite)
    pos = finite[finite >= 0]
    mids = (pos[:-1] + pos[1:]) / 2  # exact ties: must round to the even code
    for x in (mids, -mids, mids * (1 + 1e-9), mids * (1 - 1e-9)):
        ref = torch.from_numpy(x.astype(np.float32)).to(torch.float8_e4m3fn).float().numpy()
        assert np.array_equal(llama_ref.e4m3_round(x.astype(np.float32)), ref)
    assert llama_ref.e4m3_round(np.array([1000.0, -1e6]))[0] == 448.0  # saturating


def test_quantize_rows_matches_torch_recipe():
    rng = np.random.default_rng(0)
    x = llama_ref.bf16_round((rng.standard_normal((33, 512)) * 3).astype(np.float32))
    x[5] = 0.0
    x[7] *= np.float32(1e-4)
    q, s = llama_ref.quantize_rows(x)
    xt = torch.from_numpy(x)
    amax = xt.abs().amax(dim=1)
    c448 = torch.full_like(amax, 448.0)
    inv = torch.where(amax > 0, c448 / amax, torch.zeros_like(amax))
    qt = (xt * inv[:, None]).to(torch.float8_e4m3fn).float().numpy()
    assert np.array_equal(q, qt) and np.array_equal(s, (amax / c448).numpy())
    assert not q[5].any() and s[5] == 0
    err = np.abs(q * s[:, None].astype(np.float64) - x)
    assert (err <= np.abs(x).max(axis=1, keepdims=True) * 2.0 ** -4).all()


def test_fp8_presets_and_byte_accounting():
    assert QWEN_2_5_32B_FP8.weight_fp8 and not QWEN_2_5_32B.weight_fp8
    # E4M3 layer matrices take half the bytes of bf16 (+ fp32 per-channel scales); embedding / LM head stay bf16
    h, i = QWEN_2_5_32B.hidden, QWEN_2_5_32B.intermediate
    emb = 2 * 2 * QWEN_2_5_32B.vocab * h
    assert QWEN_2_5_32B_FP8.weight_bytes - emb < 0.51 * (QWEN_2_5_32B.weight_bytes - emb)
    assert LLAMA_3_3_70B_FP8.weight_bytes < 75e9  # fits one 180 GB B200 with room for the pool
    assert geometry.arena_bytes(TINY_FP8, 2048) > geometry.arena_bytes(llama_ref_tiny(), 2048)


def llama_ref_tiny():
    from paper_2505_07203_b200.config import TINY
    return TINY

"""FP8 (W8A8, E4M3) path: per-row quantisation and the kind::f8f6f4 pair GEMM against fp32 torch references.

The reference's FP8 presets (ps/presets/qwen-32b-fp8.preset:1-16, ps/presets/llama-3.3-70b-fp8.preset:1-15) only
change byte counts in its cost model; SURVEY.md §8f ranks real FP8 weights on tcgen05 kind::f8f6f4 as the next item.
Quantisation is integer-like work (a rounding of fixed inputs), so it is checked bit-exactly against torch's own
float8_e4m3fn conversion of the same fp32 products. The GEMM is floating point: its reference is the fp32 product of
the dequantised operands, with the tolerance of test_gpu_gemm (the E4M3 products are exact in the fp32 accumulator).
"""

import ctypes

import pytest

torch = pytest.importorskip("torch")

from paper_2505_07203_b200 import _lib  # noqa: E402

pytestmark = pytest.mark.gpu

TOL_BF16 = 1.5e-2
TOL_F32 = 2e-3
F8 = torch.float8_e4m3fn


def _p(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-30)).item()


def _rand(*shape, scale=1.0):
    return (torch.randn(*shape, device="cuda") * scale).to(torch.bfloat16)


def quantize(x):
    """po_op_quantize_e4m3 -> (q uint8 [R, C], scale fp32 [R])."""
    R, C = x.shape
    q = torch.empty(R, C, dtype=torch.uint8, device="cuda")
    s = torch.empty(R, dtype=torch.float32, device="cuda")
    _lib.call("po_op_quantize_e4m3", _p(x), x.stride(0), R, C, _p(q), q.stride(0), _p(s), None)
    torch.cuda.synchronize()
    return q, s


def quantize_ref(x):
    xf = x.float()
    amax = xf.abs().amax(dim=1)
    c448 = torch.full_like(amax, 448.0)  # tensor / tensor: IEEE division (a python-scalar divisor becomes a reciprocal)
    inv = torch.where(amax > 0, c448 / amax, torch.zeros_like(amax))
    return (xf * inv[:, None]).to(F8).view(torch.uint8), amax / c448


def deq(q, s):
    return q.view(F8).float() * s[:, None]


def gemm_fp8(Aq, sa, Bq, sb, out=None, resid=None, epi=_lib.EPI_BF16, rope=None, pos_offset=0, rope_cols=0):
    M, K = Aq.shape
    N = Bq.shape[0]
    ldo = out.stride(0) if out is not None else 0
    ldr = resid.stride(0) if resid is not None else 0
    _lib.call("po_op_gemm_fp8", _p(Aq), Aq.stride(0), _p(sa), _p(Bq), Bq.stride(0), _p(sb), _p(out), ldo, _p(resid),
              ldr, M, N, K, epi, _p(rope), pos_offset, rope_cols, None)
    torch.cuda.synchronize()


@pytest.mark.parametrize("R,C", [(1, 128), (7, 4096), (300, 14336), (64, 27648)])
def test_quantize_rows_bit_exact(R, C):
    torch.manual_seed(R + C)
    x = _rand(R, C, scale=3.0)
    x[0, :] *= 1e-3  # a small-magnitude row (subnormal E4M3 codes)
    if R > 2:
        x[2, :] = 0  # an all-zero row: scale 0, codes 0
    q, s = quantize(x)
    qr, sr = quantize_ref(x)
    assert torch.equal(s, sr)
    assert torch.equal(q, qr), (q != qr).sum().item()
    # round trip within half an E4M3 step (relative 2^-4) of the row maximum
    err = (deq(q, s) - x.float()).abs()
    assert (err <= x.float().abs().amax(dim=1, keepdim=True) * 2.0 ** -4 + 1e-30).all()


@pytest.mark.parametrize("M,N,K", [(128, 256, 128), (300, 512, 256), (2048, 1024, 4096), (4096, 4096, 4096),
                                   (160, 6144, 4096), (1, 4096, 4096), (150, 4096, 14336)])
def test_gemm_fp8_bf16_f32_resid(M, N, K):
    torch.manual_seed(M + N + K)
    Aq, sa = quantize(_rand(M, K))
    Bq, sb = quantize(_rand(N, K, scale=K ** -0.5))
    ref = deq(Aq, sa) @ deq(Bq, sb).T
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    gemm_fp8(Aq, sa, Bq, sb, out)
    assert _rel(out, ref) < TOL_BF16
    out32 = torch.empty(M, N, dtype=torch.float32, device="cuda")
    gemm_fp8(Aq, sa, Bq, sb, out32, epi=_lib.EPI_F32)
    assert _rel(out32, ref) < TOL_F32
    resid = torch.randn(M, N, device="cuda")
    base = resid.clone()
    gemm_fp8(Aq, sa, Bq, sb, resid=resid, epi=_lib.EPI_RESID_F32)
    assert _rel(resid, base + ref) < TOL_F32


@pytest.mark.parametrize("M", [640, 150])
def test_gemm_fp8_silu_mul(M):
    torch.manual_seed(M)
    I, K = 2048, 1024
    Aq, sa = quantize(_rand(M, K))
    gate = _rand(I, K, scale=K ** -0.5)
    up = _rand(I, K, scale=K ** -0.5)
    W = torch.stack([gate.view(I // 16, 16, K), up.view(I // 16, 16, K)], dim=1).reshape(2 * I, K).contiguous()
    Wq, sw = quantize(W)
    out = torch.empty(M, I, dtype=torch.bfloat16, device="cuda")
    gemm_fp8(Aq, sa, Wq, sw, out, epi=_lib.EPI_SILU_MUL)
    y = (deq(Aq, sa) @ deq(Wq, sw).T).view(M, I // 16, 2, 16)
    g, u = y[:, :, 0].reshape(M, I), y[:, :, 1].reshape(M, I)
    assert _rel(out, g / (1 + torch.exp(-g)) * u) < TOL_BF16


@pytest.mark.parametrize("M,K", [(300, 256), (150, 4096)])
def test_gemm_fp8_qkv_rope(M, K):
    torch.manual_seed(M + K)
    hd, nq, nkv = 128, 8, 2
    N = (nq + 2 * nkv) * hd
    Aq, sa = quantize(_rand(M, K))
    Bq, sb = quantize(_rand(N, K, scale=K ** -0.5))
    pos_offset = 1000
    pos = torch.arange(pos_offset + M, dtype=torch.float32)
    inv = 1.0 / (1e6 ** (torch.arange(0, hd, 2, dtype=torch.float32) / hd))
    ang = pos[:, None] * inv[None, :]
    table = torch.stack([torch.cos(ang), torch.sin(ang)], dim=-1).contiguous().cuda()
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    rope_cols = (nq + nkv) * hd
    gemm_fp8(Aq, sa, Bq, sb, out, epi=_lib.EPI_QKV_ROPE, rope=table, pos_offset=pos_offset, rope_cols=rope_cols)
    y = (deq(Aq, sa) @ deq(Bq, sb).T).view(M, -1, hd)
    c = table[pos_offset:pos_offset + M, :, 0][:, None, :]
    s = table[pos_offset:pos_offset + M, :, 1][:, None, :]
    x1, x2 = y[..., :64], y[..., 64:]
    rot = torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)
    ref = torch.cat([rot[:, :rope_cols // hd], y[:, rope_cols // hd:]], dim=1).reshape(M, N)
    assert _rel(out, ref) < TOL_BF16


def test_gemm_fp8_rejects_bad_shape_and_missing_scales():
    Aq, sa = quantize(_rand(64, 128))
    Bq, sb = quantize(_rand(256, 128))
    out = torch.empty(64, 256, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(_lib.PrefillOnlyError):
        _lib.call("po_op_gemm_fp8", _p(Aq), 128, None, _p(Bq), 128, _p(sb), _p(out), 256, None, 0, 64, 256, 128,
                  _lib.EPI_BF16, None, 0, 0, None)
    with pytest.raises(_lib.PrefillOnlyError):  # K % 128
        _lib.call("po_op_gemm_fp8", _p(Aq), 128, _p(sa), _p(Bq), 128, _p(sb), _p(out), 256, None, 0, 64, 256, 64,
                  _lib.EPI_BF16, None, 0, 0, None)


# ---- the FP8 engine (W8A8 layer GEMMs) against the oracle's FP8 emulation (oracle/llama_ref.py quantize_rows)
import numpy as np  # noqa: E402

from oracle import llama_ref  # noqa: E402
from paper_2505_07203_b200.config import ModelConfig, TINY_FP8  # noqa: E402
from paper_2505_07203_b200.engine import Engine  # noqa: E402

LOGIT_ATOL = 2e-2
LOGIT_RTOL = 2e-2
YES_NO = [9642, 2822]
TINY_QWEN_FP8 = ModelConfig("tiny-qwen-fp8", 2, 1280, 10, 2, 128, 1024, 32000, rms_eps=1e-6, rope_theta=1_000_000.0,
                            rope_scaling=0, qkv_bias=True, weight_fp8=True)


def tokens_for(seed, n):
    return np.random.default_rng([seed, 0, 0]).integers(0, 2 ** 32, size=n, dtype=np.uint32)


def check_fp8(model, res, toks, allowed, seed, n_cached=0):
    cfg = llama_ref.Cfg.from_model(model)
    assert cfg.weight_fp8
    logits, probs, am = llama_ref.llama_forward(cfg, llama_ref.make_weights(cfg, seed), toks, allowed)
    err = np.abs(res.logits - logits)
    tol = LOGIT_ATOL + LOGIT_RTOL * np.abs(logits)
    print(f"{model.name}: n={len(toks)} n_c={n_cached} gpu={res.logits} oracle={logits} max_err={err.max():.3e}")
    assert (err <= tol).all(), (res.logits, logits)
    srt = np.sort(logits)[::-1]
    if len(srt) > 1 and srt[0] - srt[1] > 2 * tol.max():
        assert res.index == am
    assert abs(float(res.probs.sum()) - 1.0) < 1e-5


def test_tiny_fp8_engine_matches_oracle_cold_ragged_and_hit():
    with Engine(TINY_FP8, seed=42, max_tokens=4096, chunk=1024, pool_blocks=256) as e:
        toks = tokens_for(0, 2048)
        slots = list(range(128))
        check_fp8(TINY_FP8, e.prefill(toks, YES_NO, 0, slots), toks, YES_NO, 42)
        check_fp8(TINY_FP8, e.prefill(toks, YES_NO, 1024, slots), toks, YES_NO, 42, 1024)  # prefix hit (split-K)
        for n in (1, 130):
            t = tokens_for(n, n)
            check_fp8(TINY_FP8, e.prefill(t, YES_NO), t, YES_NO, 42)


def test_qwen_style_fp8_odd_group_and_bias():
    toks = tokens_for(17, 1300)
    with Engine(TINY_QWEN_FP8, seed=5, max_tokens=2048, chunk=512, pool_blocks=128) as e:
        check_fp8(TINY_QWEN_FP8, e.prefill(toks, YES_NO), toks, YES_NO, 5)


def test_fp8_engine_load_weight_roundtrip():
    """po_load_weight on an FP8 engine quantises the given bf16 rows: loading the engine's own init reproduces it."""
    toks = tokens_for(3, 700)
    cfg = llama_ref.Cfg.from_model(TINY_FP8)
    w = llama_ref.make_weights(llama_ref.Cfg(**{**cfg.__dict__, "weight_fp8": False}), 42)  # bf16 init
    with Engine(TINY_FP8, seed=42, max_tokens=1024, chunk=512, pool_blocks=8) as e:
        before = e.prefill(toks, YES_NO).logits
        for l, lw in enumerate(w["layers"]):
            for kind, name in ((2, "wq"), (3, "wk"), (4, "wv"), (5, "wo"), (7, "w_gate"), (8, "w_up"), (9, "w_down")):
                bits = (np.ascontiguousarray(lw[name], dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)
                e.load_weight(kind, l, bits)  # bf16 bit patterns (the oracle's values are exact bf16)
        after = e.prefill(toks, YES_NO).logits
    assert np.array_equal(before, after)

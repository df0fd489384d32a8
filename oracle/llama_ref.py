"""CPU oracle for the PrefillOnly layer forward — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import this module, and only
as the checker / CPU baseline; the product path (paper_2505_07203_b200/) never calls it.

What it restates (numpy, float64 arithmetic):
  * the reference toy block (ps/numerics.py:132-171): `toy_block_forward` = block_forward_full, built
    from the same helpers the Llama forward uses (`causal_attention`, `gated_mlp`). It is PINNED against
    the reference: <= 1e-12 vs block_forward_full and the SEED42 sha256 fixture
    (pkg/tests/test_numerics.py:18,86-90), see tests/test_oracle_numerics.py.
  * the Llama-style block the B200 engine runs (embedding, RMSNorm, RoPE, GQA, residuals, allowed-row LM
    head). The reference has none of these: parity for them is UNPINNED by the reference
    and rests on the definitions stated here and in DESIGN.md, cross-checked against transformers' Llama.
  * the engine's counter-hash weight init, bit for bit (csrc/kernels.cu: unit_uniform / init kernels).

bf16-faithful: values are rounded to bf16 at the same storage points as the kernels (the folded-RMSNorm GEMM
input bf16(x . gamma), roped q/k, v, attention output, SiLU.mul output, final hidden); accumulation is float64.

FP8 (cfg.weight_fp8, the reference's FP8 presets ps/presets/qwen-32b-fp8.preset:1-16): layer weights are the bf16
init quantised per output row to E4M3, and every layer GEMM input is quantised per row the same way
(`quantize_rows`, mirroring csrc/gemm.cu quantize_rows_kernel: fp32 amax, inv = 448 / amax, e4m3 RNE satfinite of
x * inv, scale = amax / 448); products are then taken in float64 on the dequantised values.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# ------------------------------------------------------------------ bf16 and the counter hash

K_SEED = np.uint64(0x9E3779B97F4A7C15)
K_TID = np.uint64(0xD1B54A32D192ED03)
SQRT3_F32 = np.float32(1.7320508)
TID_EMBED, TID_FINAL_NORM, TID_LM_HEAD = 0xFFFF0, 0xFFFF1, 0xFFFF2
K_ATTN_NORM, K_Q, K_K, K_V, K_O, K_MLP_NORM, K_GATE, K_UP, K_DOWN, K_QKV_BIAS = range(10)


def bf16_round(x) -> np.ndarray:
    """Round float32 values to the nearest bf16 (ties to even); returns float32 holding bf16 values."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    bits = a.view(np.uint32).astype(np.uint64)
    rounded = ((bits + np.uint64(0x7FFF) + ((bits >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)) << np.uint64(16)
    return rounded.astype(np.uint32).view(np.float32).reshape(a.shape)


def e4m3_round(x) -> np.ndarray:
    """Round to the nearest E4M3 value (OCP FP8, ties to even, saturating at +-448); float64 in, float64 out."""
    a = np.asarray(x, dtype=np.float64)
    m = np.minimum(np.abs(a), 448.0)
    _, ex = np.frexp(m)                      # m = f * 2^ex, f in [0.5, 1)
    e = np.maximum(ex - 1, -6)               # binade exponent; subnormals share the 2^-6 binade's spacing
    step = np.ldexp(1.0, e - 3)              # 3 mantissa bits
    return np.sign(a) * np.rint(m / step) * step


def quantize_rows(x) -> tuple[np.ndarray, np.ndarray]:
    """Per-row E4M3 quantisation as the kernel does it in fp32: returns (codes as float64, scale float32)."""
    xf = np.asarray(x, dtype=np.float32)
    amax = np.abs(xf).max(axis=-1).astype(np.float32)
    with np.errstate(divide="ignore"):
        inv = np.where(amax > 0, np.float32(448.0) / amax, np.float32(0.0)).astype(np.float32)
    y = (xf * inv[..., None]).astype(np.float32)
    return e4m3_round(y), (amax / np.float32(448.0)).astype(np.float32)


def fp8_dequant_rows(x) -> np.ndarray:
    """quantize_rows then dequantise (codes * scale) in float64: the value an FP8 GEMM multiplies."""
    q, sc = quantize_rows(x)
    return q * sc.astype(np.float64)[..., None]


def splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def unit_uniform(seed: int, tid: int, idx: np.ndarray) -> np.ndarray:
    """Counter-based U[-sqrt3, sqrt3) in float32, identical to csrc/kernels.cu:unit_uniform."""
    with np.errstate(over="ignore"):
        key = np.uint64(seed) * K_SEED + np.uint64(tid) * K_TID + idx.astype(np.uint64)
    z = splitmix64(key)
    u = (z >> np.uint64(40)).astype(np.float32) * np.float32(1.0 / 16777216.0)
    return ((np.float32(2.0) * u - np.float32(1.0)) * SQRT3_F32).astype(np.float32)


def fan_scale(fan_in: int) -> np.float32:
    return np.float32(1.0 / np.sqrt(np.float64(fan_in)))


def init_matrix(seed: int, tid: int, rows: int, cols: int, scale) -> np.ndarray:
    """bf16 weight [rows, cols] (as float32) = bf16(u * scale) (init_bf16_kernel, INIT_PLAIN)."""
    out = np.empty((rows, cols), dtype=np.float32)
    step = max(1, (1 << 22) // cols)
    for r0 in range(0, rows, step):
        r1 = min(rows, r0 + step)
        idx = np.arange(r0 * cols, r1 * cols, dtype=np.uint64)
        out[r0:r1] = bf16_round(unit_uniform(seed, tid, idx) * np.float32(scale)).reshape(r1 - r0, cols)
    return out


class LazyRows:
    """Rows of a counter-hash bf16 matrix generated on demand (`m[idx]` == init_matrix(...)[idx]), for the vocab-sized
    embedding / LM head at full model size: a request touches only its token rows and the allowed rows."""

    def __init__(self, seed: int, tid: int, rows: int, cols: int, scale):
        self.seed, self.tid, self.rows, self.cols, self.scale = seed, tid, rows, cols, np.float32(scale)

    def __getitem__(self, idx) -> np.ndarray:
        idx = np.atleast_1d(np.asarray(idx, dtype=np.int64))
        if idx.size and (idx.min() < 0 or idx.max() >= self.rows):
            raise IndexError("row out of range")
        out = np.empty((idx.size, self.cols), dtype=np.float32)
        col = np.arange(self.cols, dtype=np.uint64)
        step = max(1, (1 << 22) // self.cols)
        for r0 in range(0, idx.size, step):
            sel = idx[r0:r0 + step].astype(np.uint64)
            flat = (sel[:, None] * np.uint64(self.cols) + col[None, :]).ravel()
            out[r0:r0 + sel.size] = bf16_round(unit_uniform(self.seed, self.tid, flat) * self.scale).reshape(-1, self.cols)
        return out


def init_norm(seed: int, tid: int, n: int) -> np.ndarray:
    u = unit_uniform(seed, tid, np.arange(n, dtype=np.uint64))
    return bf16_round(np.float32(1.0) + np.float32(0.05) * u)


def init_bias(seed: int, tid: int, n: int) -> np.ndarray:
    """bf16(0.1 * u) (init_bias_kernel)."""
    return bf16_round(np.float32(0.1) * unit_uniform(seed, tid, np.arange(n, dtype=np.uint64)))


def layer_tid(layer: int, kind: int) -> int:
    return layer * 16 + kind


# ------------------------------------------------------------------ configuration and weights


@dataclass(frozen=True)
class Cfg:
    num_layers: int
    hidden: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    intermediate: int
    vocab: int
    rms_eps: float = 1e-5
    rope_theta: float = 500_000.0
    rope_scaling: int = 1
    rope_factor: float = 8.0
    rope_low_freq_factor: float = 1.0
    rope_high_freq_factor: float = 4.0
    rope_original_max_pos: int = 8192
    qkv_bias: bool = False
    weight_fp8: bool = False

    @classmethod
    def from_model(cls, m) -> "Cfg":
        return cls(**{k: getattr(m, k) for k in cls.__dataclass_fields__})


def make_weights(cfg: Cfg, seed: int, lazy_vocab: bool = False) -> dict:
    """All weights as float32 arrays holding bf16 values, in the logical (un-interleaved) layout.

    lazy_vocab: the embedding and LM head become LazyRows (same values, generated per indexed row)."""
    h, i_, hd = cfg.hidden, cfg.intermediate, cfg.head_dim
    mat = LazyRows if lazy_vocab else init_matrix
    w = {
        "embed": mat(seed, TID_EMBED, cfg.vocab, h, np.float32(1.0)),
        "lm_head": mat(seed, TID_LM_HEAD, cfg.vocab, h, fan_scale(h)),
        "final_norm": init_norm(seed, TID_FINAL_NORM, h),
        "layers": [],
    }
    for l in range(cfg.num_layers):
        w["layers"].append({
            "attn_norm": init_norm(seed, layer_tid(l, K_ATTN_NORM), h),
            "wq": init_matrix(seed, layer_tid(l, K_Q), cfg.n_heads * hd, h, fan_scale(h)),
            "wk": init_matrix(seed, layer_tid(l, K_K), cfg.n_kv_heads * hd, h, fan_scale(h)),
            "wv": init_matrix(seed, layer_tid(l, K_V), cfg.n_kv_heads * hd, h, fan_scale(h)),
            "wo": init_matrix(seed, layer_tid(l, K_O), h, cfg.n_heads * hd, fan_scale(cfg.n_heads * hd)),
            "mlp_norm": init_norm(seed, layer_tid(l, K_MLP_NORM), h),
            "w_gate": init_matrix(seed, layer_tid(l, K_GATE), i_, h, fan_scale(h)),
            "w_up": init_matrix(seed, layer_tid(l, K_UP), i_, h, fan_scale(h)),
            "w_down": init_matrix(seed, layer_tid(l, K_DOWN), h, i_, fan_scale(i_)),
        })
        if cfg.qkv_bias:
            w["layers"][-1]["bqkv"] = init_bias(seed, layer_tid(l, K_QKV_BIAS), (cfg.n_heads + 2 * cfg.n_kv_heads) * hd)
        if cfg.weight_fp8:  # E4M3 per output row (rows are independent, so q/k/v and gate/up quantise separately)
            for name in ("wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down"):
                w["layers"][-1][name] = fp8_dequant_rows(w["layers"][-1][name])
    return w


# ------------------------------------------------------------------ shared block pieces


def silu(z: np.ndarray) -> np.ndarray:
    """z / (1 + e^-z)  (ps/numerics.py:123-124)."""
    return z / (1.0 + np.exp(-z))


def causal_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, q_offset: int = 0) -> np.ndarray:
    """Causal softmax(q k^T / sqrt(d)) v per head, GQA by head grouping (ps/numerics.py:132-146).

    q: (n_q, Hq, d); k, v: (n_kv, Hkv, d); query row r sits at position q_offset + r and attends to keys
    0..q_offset+r (the triu mask of the reference shifted by the cached prefix).
    """
    n_q, hq, d = q.shape
    n_kv, hkv, _ = k.shape
    group = hq // hkv
    pos = np.arange(q_offset, q_offset + n_q)
    keys = np.arange(n_kv)
    masked = keys[None, :] > pos[:, None]
    out = np.empty((n_q, hq, d), dtype=np.float64)
    for hh in range(hq):
        kh = k[:, hh // group, :].astype(np.float64)
        vh = v[:, hh // group, :].astype(np.float64)
        s = (q[:, hh, :].astype(np.float64) @ kh.T) / np.sqrt(d)
        s[masked] = -np.inf
        s -= s.max(axis=1, keepdims=True)
        np.exp(s, out=s)
        s /= s.sum(axis=1, keepdims=True)
        out[:, hh, :] = s @ vh
    return out


def gated_mlp(x: np.ndarray, w_gate: np.ndarray, w_up: np.ndarray, w_down: np.ndarray, round_act=False):
    """silu(x Wg) * (x Wu) then Wd, weights given as [in, out] (ps/numerics.py:165-170)."""
    g = x @ w_gate
    u = x @ w_up
    act = silu(g) * u
    if round_act:
        act = bf16_round(act).astype(np.float64)
    return act @ w_down


# ------------------------------------------------------------------ reference toy block (pinned)


def toy_block_forward(w_qkv: np.ndarray, w_out: np.ndarray, w_gate_up: np.ndarray, w_down: np.ndarray,
                      x: np.ndarray) -> np.ndarray:
    """block_forward_full (ps/numerics.py:149-171): single-head causal attention + SiLU-gated MLP.

    Weights in the reference's [in, out] layout; [q|k|v] and [gate|up] column splits (:143, :168).
    """
    h = w_qkv.shape[0]
    inter = w_down.shape[0]
    qkv = x @ w_qkv
    q, k, v = qkv[:, :h], qkv[:, h:2 * h], qkv[:, 2 * h:]
    ctx = causal_attention(q[:, None, :], k[:, None, :], v[:, None, :])[:, 0, :]
    attn = ctx @ w_out
    return gated_mlp(attn, w_gate_up[:, :inter], w_gate_up[:, inter:], w_down)


# ------------------------------------------------------------------ Llama block (engine semantics)


def rope_inv_freq(cfg: Cfg) -> np.ndarray:
    """Llama-3 RoPE inverse frequencies, float64 then rounded once to float32 (engine.cu:rope_inv_freq)."""
    i = np.arange(cfg.head_dim // 2, dtype=np.float64)
    f = 1.0 / np.power(np.float64(np.float32(cfg.rope_theta)), 2.0 * i / cfg.head_dim)
    if cfg.rope_scaling == 1:
        factor = np.float64(np.float32(cfg.rope_factor))
        low = np.float64(np.float32(cfg.rope_low_freq_factor))
        high = np.float64(np.float32(cfg.rope_high_freq_factor))
        orig = np.float64(cfg.rope_original_max_pos)
        low_wl, high_wl = orig / low, orig / high
        wl = 2.0 * np.pi / f
        smooth = (orig / wl - low) / (high - low)
        mid = (1.0 - smooth) * f / factor + smooth * f
        f = np.where(wl > low_wl, f / factor, np.where(wl >= high_wl, mid, f))
    return f.astype(np.float32)


def rope_table(cfg: Cfg, n: int) -> tuple[np.ndarray, np.ndarray]:
    inv = rope_inv_freq(cfg)
    ang = np.arange(n, dtype=np.float32)[:, None] * inv[None, :]  # float32 product
    a64 = ang.astype(np.float64)
    return np.cos(a64).astype(np.float32), np.sin(a64).astype(np.float32)


def rmsnorm(x: np.ndarray, gamma: np.ndarray, eps: float, rnd=None) -> np.ndarray:
    ms = np.mean(x * x, axis=-1, keepdims=True)
    y = (x / np.sqrt(ms + eps)) * gamma
    return (rnd or _round64)(y)


def _round64(x):
    return bf16_round(x).astype(np.float64)


def _exact(x):
    return np.asarray(x, dtype=np.float64)


def folded_norm(x: np.ndarray, gamma: np.ndarray, eps: float, rnd) -> tuple[np.ndarray, np.ndarray]:
    """The engine's RMSNorm, folded across the next GEMM: returns (rnd(x . gamma), 1/rms per row); the GEMM
    output row is multiplied by 1/rms (csrc/gemm.cu row_inv_rms). Exact algebra equals rnd-free rmsnorm."""
    inv = 1.0 / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)
    return rnd(x * gamma), inv


def apply_rope(x: np.ndarray, cos: np.ndarray, sin: np.ndarray) -> np.ndarray:
    """Rotate-half RoPE on (n, H, d): pairs (i, i + d/2)."""
    half = x.shape[-1] // 2
    c = cos[:, None, :].astype(np.float64)
    s = sin[:, None, :].astype(np.float64)
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def llama_forward(cfg: Cfg, w: dict, tokens, allowed, n_cached: int = 0, return_hidden: bool = False,
                  round_bf16: bool = True):
    """Prefill-only forward of one request; returns (logits, probs, argmax) over the allowed ids.

    Cached-prefix rows only serve as keys; their K/V equal what a cold forward computes (causality), so the
    oracle computes them directly. Layer semantics follow engine.cu's header comment.
    """
    toks = np.asarray(tokens, dtype=np.uint64) % np.uint64(cfg.vocab)
    n = len(toks)
    hd, hq, hkv = cfg.head_dim, cfg.n_heads, cfg.n_kv_heads
    cos, sin = rope_table(cfg, n)
    R = _round64 if round_bf16 else _exact
    if not round_bf16:  # exact float64 Llama (for the transformers cross-check): exact RoPE angles too
        inv = rope_inv_freq(cfg).astype(np.float64)
        ang = np.arange(n, dtype=np.float64)[:, None] * inv[None, :]
        cos, sin = np.cos(ang), np.sin(ang)
    x = w["embed"][toks.astype(np.int64)].astype(np.float64)
    # FP8: every layer GEMM input is quantised per row (after its bf16 rounding), the weights already are
    Q = fp8_dequant_rows if getattr(cfg, "weight_fp8", False) else (lambda a: a)
    for lw in w["layers"]:
        xg, inv = folded_norm(x, lw["attn_norm"], cfg.rms_eps, R)
        xg = Q(xg)
        q = inv * (xg @ lw["wq"].T.astype(np.float64))
        k = inv * (xg @ lw["wk"].T.astype(np.float64))
        v = inv * (xg @ lw["wv"].T.astype(np.float64))
        if "bqkv" in lw:  # Qwen2: bias added to the projections before RoPE
            b = lw["bqkv"].astype(np.float64)
            q, k, v = q + b[: hq * hd], k + b[hq * hd:(hq + hkv) * hd], v + b[(hq + hkv) * hd:]
        q, k, v = q.reshape(n, hq, hd), k.reshape(n, hkv, hd), v.reshape(n, hkv, hd)
        q = R(apply_rope(q, cos, sin))
        k = R(apply_rope(k, cos, sin))
        v = R(v)
        ctx = Q(R(causal_attention(q, k, v)).reshape(n, hq * hd))
        x = x + ctx @ lw["wo"].T.astype(np.float64)
        xg2, inv2 = folded_norm(x, lw["mlp_norm"], cfg.rms_eps, R)
        xg2 = Q(xg2)
        g = inv2 * (xg2 @ lw["w_gate"].T.astype(np.float64))
        u = inv2 * (xg2 @ lw["w_up"].T.astype(np.float64))
        act = Q(R(silu(g) * u))
        x = x + act @ lw["w_down"].T.astype(np.float64)
    h_last = rmsnorm(x[-1:], w["final_norm"], cfg.rms_eps, R)[0]
    alw = np.asarray(allowed, dtype=np.int64)
    logits = w["lm_head"][alw].astype(np.float64) @ h_last
    e = np.exp(logits - logits.max())
    probs = e / e.sum()
    if return_hidden:
        return logits, probs, int(np.argmax(logits)), x
    return logits, probs, int(np.argmax(logits))

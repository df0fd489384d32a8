"""KV-manager sizing: bytes per token, peak prefill memory per mode, maximum input length, prefix capacity.

The reference computes these in closed form with a calibrated activation factor (ps/geometry.py:147-230,
act_overhead_factor). Here the hybrid mode is the engine's *actual* allocation (csrc/engine.cu po_init:
fp32 residual, bf16 normed/ctx buffer, the one-layer qkv buffer, one MLP chunk, the RoPE table, split
workspaces), so `arena_bytes` equals what po_engine_info reports (tests/test_gpu_engine.py), and the
"profile run" is that arena plus the weights; the prefix pool gets what HBM has left.
The FULL / KV_DISCARD / CHUNKED modes keep the reference's definitions for comparison.
"""

from __future__ import annotations

import math

from .config import DEFAULT_CHUNK, ModelConfig

FULL, KV_DISCARD, CHUNKED, HYBRID = "full", "kv-discard", "chunked", "hybrid"
B200_HBM_BYTES = 183_359 * 2 ** 20  # nvidia-smi total memory of a B200


class GeometryError(ValueError):
    pass


def kv_bytes_per_token(m: ModelConfig) -> tuple[int, int]:
    """(per-layer, all-layer) bf16 K/V bytes per token (ps/geometry.py:147-150)."""
    return m.kv_bytes_per_token


def intermediate_bytes_per_token(m: ModelConfig) -> int:
    """gate/up output bytes per token, the MLP's activation spike (ps/geometry.py:153-159), bf16."""
    return 2 * m.intermediate * 2


def arena_bytes(m: ModelConfig, max_tokens: int, chunk: int = DEFAULT_CHUNK) -> int:
    """Activation arena po_init allocates for `max_tokens` (hybrid prefill, one layer of K/V).

    Mirrors csrc/engine.cu: resid fp32 [T,h] + ctx bf16 [T,max(h,Hq*d)] + qkv bf16 [T,(Hq+2Hkv)*d]
    + xg bf16 [T,h] + sum-of-squares fp32 2 x [T, h/128]
    + MLP chunk bf16 [min(chunk,T), I] + RoPE (cos,sin) fp32 [T, d/2] + per-request staging; the split-KV /
    split-K workspaces (short queries only) are excluded and bounded separately.
    """
    T = max_tokens
    h, hd = m.hidden, m.head_dim
    ctx = m.n_heads * hd
    qkvc = (m.n_heads + 2 * m.n_kv_heads) * hd
    rows = min(chunk, T)
    b = 4 * T * h + 2 * T * max(h, ctx) + 2 * T * qkvc + 2 * rows * m.intermediate + 8 * T * (hd // 2)
    b += 2 * T * h + 2 * 4 * T * (h // 128)  # folded-RMSNorm input xg (bf16) + two sum-of-squares buffers
    if m.weight_fp8:  # E4M3 copies of the GEMM inputs (xg, ctx, act) + their per-row scales
        b += T * h + T * ctx + rows * m.intermediate + 4 * (2 * T + rows)
    max_blocks = T // 16 + 1
    # token ids, a 4-entry ring of (cached-slot, admission-slot) block tables, allowed ids, logits, probs, argmax
    b += 4 * T + 4 * (4 * max_blocks + 4 * max_blocks) + 3 * 4 * m.vocab + 16
    return b


def peak_prefill_memory(m: ModelConfig, n: int, mode: str = HYBRID, chunk: int = DEFAULT_CHUNK) -> int:
    """Peak bytes to prefill n tokens. HYBRID = this engine's arena; the others follow ps/geometry.py:162-183
    with the engine's activation footprint (no calibration factor)."""
    if n <= 0:
        raise GeometryError("n must be positive")
    kv_layer, kv_total = kv_bytes_per_token(m)
    if mode == HYBRID:
        return m.weight_bytes + arena_bytes(m, n, chunk)
    act_full = 4 * n * m.hidden + 2 * n * m.hidden + intermediate_bytes_per_token(m) * n
    act_chunk = 4 * n * m.hidden + 2 * n * m.hidden + intermediate_bytes_per_token(m) * min(n, chunk)
    if mode == FULL:
        return m.weight_bytes + kv_total * n + act_full
    if mode == KV_DISCARD:
        return m.weight_bytes + kv_layer * n + act_full
    if mode == CHUNKED:
        return m.weight_bytes + kv_total * n + act_chunk
    raise GeometryError(f"unknown mode {mode!r}")


def largest_fitting(peak_fn, budget: int) -> int:
    """Largest n >= 0 with peak_fn(n) <= budget for nondecreasing peak_fn (ps/geometry.py:186-200)."""
    if peak_fn(1) > budget:
        return 0
    lo, hi = 1, 2
    while peak_fn(hi) <= budget:
        lo, hi = hi, hi * 2
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if peak_fn(mid) <= budget:
            lo = mid
        else:
            hi = mid
    return lo


def max_input_length(m: ModelConfig, hbm_bytes: int = B200_HBM_BYTES, mode: str = HYBRID,
                     chunk: int = DEFAULT_CHUNK, reserve_bytes: int = 2 << 30) -> int:
    """MIL on one GPU with `reserve_bytes` kept for the CUDA context (ps/geometry.py:203-212)."""
    budget = hbm_bytes - reserve_bytes
    if budget < m.weight_bytes:
        raise GeometryError(f"{m.name}: weights do not fit")
    return largest_fitting(lambda n: peak_prefill_memory(m, n, mode, chunk), budget)


def prefix_cache_capacity(m: ModelConfig, user_mil: int, hbm_bytes: int = B200_HBM_BYTES,
                          chunk: int = DEFAULT_CHUNK, reserve_bytes: int = 2 << 30) -> int:
    """Prefix-pool tokens left after reserving the hybrid working set for user_mil (ps/geometry.py:215-230)."""
    limit = max_input_length(m, hbm_bytes, HYBRID, chunk, reserve_bytes)
    if user_mil > limit:
        raise GeometryError(f"user_mil {user_mil} exceeds hybrid MIL {limit}")
    free = hbm_bytes - reserve_bytes - peak_prefill_memory(m, user_mil, HYBRID, chunk)
    _, kv_total = kv_bytes_per_token(m)
    return max(0, free // kv_total)


def peak_ratio(m: ModelConfig, n: int, chunk: int = DEFAULT_CHUNK) -> float:
    """Hybrid over full activation+KV footprint (excluding weights): the reference's peak_ratio
    (ps/numerics.py:278-282) at model scale."""
    full = peak_prefill_memory(m, n, FULL) - m.weight_bytes
    hyb = peak_prefill_memory(m, n, HYBRID, chunk) - m.weight_bytes
    return hyb / full if full else math.nan

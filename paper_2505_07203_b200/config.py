"""Model shapes and engine sizing.

The reference's ModelGeometry (ps/geometry.py:26-57) and its presets
(ps/presets/llama-3.1-8b.preset:7-15, qwen-32b-fp8.preset:7-16) carry only the byte-arithmetic
fields. A real forward also needs query heads, vocabulary, RMSNorm epsilon and RoPE constants; those
come from the public model configs and are stated here (parity for them is unpinned).
"""

from __future__ import annotations

import ctypes
from dataclasses import asdict, dataclass, replace

DEFAULT_CHUNK = 8192  # ps/geometry.py:14
BLOCK_TOKENS = 16  # CacheConfig.block_tokens default, ps/cache.py:65-80


@dataclass(frozen=True)
class ModelConfig:
    name: str
    num_layers: int
    hidden: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    intermediate: int
    vocab: int
    rms_eps: float = 1e-5
    rope_theta: float = 500_000.0
    rope_scaling: int = 1  # 0 none, 1 llama3
    rope_factor: float = 8.0
    rope_low_freq_factor: float = 1.0
    rope_high_freq_factor: float = 4.0
    rope_original_max_pos: int = 8192
    qkv_bias: bool = False  # Qwen2-style q/k/v projection bias
    weight_fp8: bool = False  # E4M3 layer weights + per-channel scales, W8A8 GEMMs (the reference's FP8 presets)

    @property
    def kv_bytes_per_token(self) -> tuple[int, int]:
        """(per-layer, all-layer) bf16 K/V bytes of one token (ps/geometry.py:147-150)."""
        per_layer = 2 * self.n_kv_heads * self.head_dim * 2
        return per_layer, per_layer * self.num_layers

    @property
    def weight_bytes(self) -> int:
        h, i = self.hidden, self.intermediate
        qkv = (self.n_heads + 2 * self.n_kv_heads) * self.head_dim * h
        o = self.n_heads * self.head_dim * h
        if self.weight_fp8:  # E4M3 matrices + fp32 per-output-channel scales; embedding, LM head, norms bf16
            qkv_rows = (self.n_heads + 2 * self.n_kv_heads) * self.head_dim
            per_layer = qkv + o + 3 * h * i + 4 * (qkv_rows + h + 2 * i + h) + 2 * 2 * h
            return self.num_layers * per_layer + 2 * (2 * self.vocab * h + h)
        per_layer = qkv + o + 3 * h * i + 2 * h
        return 2 * (self.num_layers * per_layer + 2 * self.vocab * h + h)

    def linear_flops_per_token(self) -> float:
        """Dense-layer FLOPs per token over all layers (ps/costs.py:126-131)."""
        h = self.hidden
        q_dim = self.n_heads * self.head_dim
        kv_dim = self.n_kv_heads * self.head_dim
        # reference formula (ps/costs.py:126-131) assumes q_dim == h; stated generally here (equal for Llama/Qwen)
        per_layer = 2.0 * (h * (q_dim + 2 * kv_dim) + q_dim * h + 3 * h * self.intermediate)
        return self.num_layers * per_layer

    def attn_flops_per_pair(self) -> float:
        """Attention FLOPs per (query, key) pair over all layers (ps/costs.py:134-136)."""
        return 4.0 * self.hidden * self.num_layers

    def request_flops(self, n: int, n_cached: int = 0, n_allowed: int = 2) -> float:
        """Algorithmic FLOPs of one request: linear x miss + attn x (n^2 - n_c^2)/2 (ps/costs.py:275-277)."""
        miss = n - n_cached
        pairs = (n * n - n_cached * n_cached) / 2.0
        return self.linear_flops_per_token() * miss + self.attn_flops_per_pair() * pairs + 2.0 * self.hidden * n_allowed


# Llama-3.1-8B: meta-llama/Llama-3.1-8B config.json (rope_scaling llama3, factor 8, theta 5e5, eps 1e-5)
LLAMA_3_1_8B = ModelConfig("llama-3.1-8b", 32, 4096, 32, 8, 128, 14336, 128_256)
# Tiny parity config (BASELINE.json configs[0]): 2 layers, d=256, GQA 2:1, build-chosen and stated.
TINY = ModelConfig("tiny", 2, 256, 2, 1, 128, 1024, 32_000)
# Qwen-2.5-32B shapes (Qwen/Qwen2.5-32B config.json): rope theta 1e6, eps 1e-6, no rope scaling, q/k/v
# bias. 40 query / 8 kv heads is an odd GQA group (5): attention runs two query blocks of one head per CTA.
QWEN_2_5_32B = ModelConfig("qwen-2.5-32b", 64, 5120, 40, 8, 128, 27648, 152_064, rms_eps=1e-6,
                           rope_theta=1_000_000.0, rope_scaling=0, qkv_bias=True)

# The reference's FP8-weight presets (ps/presets/qwen-32b-fp8.preset:1-16, ps/presets/llama-3.3-70b-fp8.preset:1-15):
# the same shapes with E4M3 layer weights. Llama-3.3-70B: meta-llama/Llama-3.3-70B-Instruct config.json.
QWEN_2_5_32B_FP8 = replace(QWEN_2_5_32B, name="qwen-2.5-32b-fp8", weight_fp8=True)
LLAMA_3_3_70B_FP8 = ModelConfig("llama-3.3-70b-fp8", 80, 8192, 64, 8, 128, 28672, 128_256, weight_fp8=True)
TINY_FP8 = replace(TINY, name="tiny-fp8", weight_fp8=True)

PRESETS = {c.name: c for c in (TINY, LLAMA_3_1_8B, QWEN_2_5_32B, QWEN_2_5_32B_FP8, LLAMA_3_3_70B_FP8, TINY_FP8)}


def get_preset(name: str) -> ModelConfig:
    try:
        return PRESETS[name]
    except KeyError:
        raise ValueError(f"unknown model preset {name!r}; known: {sorted(PRESETS)}") from None


class PoModelCfg(ctypes.Structure):
    """ctypes mirror of po_model_cfg (include/prefillonly.h)."""

    _fields_ = [
        ("num_layers", ctypes.c_int32),
        ("hidden", ctypes.c_int32),
        ("n_heads", ctypes.c_int32),
        ("n_kv_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("intermediate", ctypes.c_int32),
        ("vocab", ctypes.c_int32),
        ("rms_eps", ctypes.c_float),
        ("rope_theta", ctypes.c_float),
        ("rope_scaling", ctypes.c_int32),
        ("rope_factor", ctypes.c_float),
        ("rope_low_freq_factor", ctypes.c_float),
        ("rope_high_freq_factor", ctypes.c_float),
        ("rope_original_max_pos", ctypes.c_int32),
        ("max_tokens", ctypes.c_int32),
        ("chunk", ctypes.c_int32),
        ("block_tokens", ctypes.c_int32),
        ("pool_blocks", ctypes.c_int64),
        ("pool_mem_fraction", ctypes.c_double),
        ("last_row_only", ctypes.c_int32),
        ("qkv_bias", ctypes.c_int32),
        ("weight_fp8", ctypes.c_int32),
    ]


def to_c_cfg(model: ModelConfig, max_tokens: int, chunk: int = DEFAULT_CHUNK, block_tokens: int = BLOCK_TOKENS,
             pool_blocks: int = -1, pool_mem_fraction: float = 0.9, last_row_only: bool = True) -> PoModelCfg:
    d = asdict(model)
    d.pop("name")
    d["qkv_bias"] = int(d["qkv_bias"])
    d["weight_fp8"] = int(d["weight_fp8"])
    return PoModelCfg(**d, max_tokens=max_tokens, chunk=chunk, block_tokens=block_tokens, pool_blocks=pool_blocks,
                      pool_mem_fraction=pool_mem_fraction, last_row_only=int(last_row_only))


def executed_flops(model: ModelConfig, n: int, n_cached: int = 0, last_row_only: bool = True) -> float:
    """FLOPs the engine actually executes: with last_row_only the last layer runs attention, O-proj and the
    MLP for the final row only (its K/V are still computed for every row)."""
    full = model.request_flops(n, n_cached)
    if not last_row_only:
        return full
    h, i_ = model.hidden, model.intermediate
    L = model.num_layers
    miss = n - n_cached
    rows_skipped = max(0, miss - 1)
    o_mlp_per_row = 2.0 * h * (model.n_heads * model.head_dim) + 6.0 * h * i_
    attn_layer = model.attn_flops_per_pair() / L * (n * n - n_cached * n_cached) / 2.0
    attn_last_row = model.attn_flops_per_pair() / L * n
    return full - rows_skipped * o_mlp_per_row - (attn_layer - attn_last_row)


__all__ = ["ModelConfig", "PoModelCfg", "to_c_cfg", "get_preset", "PRESETS", "TINY", "LLAMA_3_1_8B",
           "QWEN_2_5_32B", "QWEN_2_5_32B_FP8", "LLAMA_3_3_70B_FP8", "TINY_FP8", "DEFAULT_CHUNK", "BLOCK_TOKENS", "replace"]

"""Pins for the parts of the Llama block the reference does not define (parity unpinned).

* bf16 rounding vs torch's bfloat16 conversion;
* RoPE llama3 inverse frequencies vs transformers' implementation;
* the whole oracle forward (with bf16 rounding disabled) vs transformers' LlamaForCausalLM in float64,
  using the oracle's counter-hash weights.
"""

import numpy as np
import pytest

from oracle import llama_ref
from paper_2505_07203_b200.config import LLAMA_3_1_8B, TINY

torch = pytest.importorskip("torch")


def test_bf16_round_matches_torch():
    x = np.random.default_rng(0).normal(size=100_000).astype(np.float32) * 37
    x[:4] = [0.0, -0.0, 1e-40, 3.0e38]
    mine = llama_ref.bf16_round(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float32).numpy()
    assert np.array_equal(mine, ref)


def test_hash_uniform_moments_and_determinism():
    idx = np.arange(1_000_000, dtype=np.uint64)
    u = llama_ref.unit_uniform(3, 17, idx)
    assert np.array_equal(u, llama_ref.unit_uniform(3, 17, idx))
    assert abs(u.mean()) < 5e-3 and abs(u.std() - 1.0) < 5e-3
    assert u.min() >= -np.float32(1.7320508) and u.max() < np.float32(1.7320508)
    assert not np.array_equal(u[:100], llama_ref.unit_uniform(3, 18, idx[:100]))


def test_rope_inv_freq_matches_transformers_llama3():
    tr = pytest.importorskip("transformers")
    from transformers.modeling_rope_utils import ROPE_INIT_FUNCTIONS

    cfg = tr.LlamaConfig(hidden_size=4096, num_attention_heads=32, num_key_value_heads=8, head_dim=128,
                         rope_theta=500000.0, max_position_embeddings=131072,
                         rope_scaling={"rope_type": "llama3", "factor": 8.0, "low_freq_factor": 1.0,
                                       "high_freq_factor": 4.0, "original_max_position_embeddings": 8192})
    inv, _ = ROPE_INIT_FUNCTIONS["llama3"](cfg, "cpu")
    mine = llama_ref.rope_inv_freq(llama_ref.Cfg.from_model(LLAMA_3_1_8B))
    # transformers computes in fp32 arithmetic, the oracle in fp64 rounded once: agree to fp32 ulps
    assert np.allclose(mine, inv.numpy(), rtol=2e-6, atol=0)


def _hf_llama(cfg: llama_ref.Cfg, w):
    tr = pytest.importorskip("transformers")
    hc = tr.LlamaConfig(vocab_size=cfg.vocab, hidden_size=cfg.hidden, intermediate_size=cfg.intermediate,
                        num_hidden_layers=cfg.num_layers, num_attention_heads=cfg.n_heads,
                        num_key_value_heads=cfg.n_kv_heads, head_dim=cfg.head_dim, rms_norm_eps=cfg.rms_eps,
                        rope_theta=cfg.rope_theta, max_position_embeddings=131072, tie_word_embeddings=False,
                        rope_scaling={"rope_type": "llama3", "factor": cfg.rope_factor,
                                      "low_freq_factor": cfg.rope_low_freq_factor,
                                      "high_freq_factor": cfg.rope_high_freq_factor,
                                      "original_max_position_embeddings": cfg.rope_original_max_pos},
                        attention_bias=False, mlp_bias=False)
    hc._attn_implementation = "eager"
    m = tr.LlamaForCausalLM(hc).double().eval()
    t = lambda a: torch.from_numpy(np.asarray(a, dtype=np.float64))
    with torch.no_grad():
        m.model.embed_tokens.weight.copy_(t(w["embed"]))
        m.lm_head.weight.copy_(t(w["lm_head"]))
        m.model.norm.weight.copy_(t(w["final_norm"]))
        for l, lw in enumerate(w["layers"]):
            L = m.model.layers[l]
            L.input_layernorm.weight.copy_(t(lw["attn_norm"]))
            L.post_attention_layernorm.weight.copy_(t(lw["mlp_norm"]))
            L.self_attn.q_proj.weight.copy_(t(lw["wq"]))
            L.self_attn.k_proj.weight.copy_(t(lw["wk"]))
            L.self_attn.v_proj.weight.copy_(t(lw["wv"]))
            L.self_attn.o_proj.weight.copy_(t(lw["wo"]))
            L.mlp.gate_proj.weight.copy_(t(lw["w_gate"]))
            L.mlp.up_proj.weight.copy_(t(lw["w_up"]))
            L.mlp.down_proj.weight.copy_(t(lw["w_down"]))
    return m


def test_oracle_forward_matches_transformers_llama_f64():
    cfg = llama_ref.Cfg.from_model(TINY)
    w = llama_ref.make_weights(cfg, 42)
    toks = np.random.default_rng([1, 0, 0]).integers(0, 2 ** 32, size=300, dtype=np.uint32)
    allowed = [9642, 2822, 17, 31999]
    logits, probs, am = llama_ref.llama_forward(cfg, w, toks, allowed, round_bf16=False)
    m = _hf_llama(cfg, w)
    ids = torch.from_numpy((toks % cfg.vocab).astype(np.int64))[None]
    with torch.no_grad():
        hf = m(input_ids=ids).logits[0, -1].numpy()
    # transformers evaluates RoPE angles/cos/sin in fp32 even for a float64 model: agreement to ~1e-7
    assert np.allclose(logits, hf[allowed], rtol=1e-5, atol=1e-5)
    assert am == int(np.argmax(hf[allowed]))


def test_bf16_faithful_forward_close_to_exact():
    cfg = llama_ref.Cfg.from_model(TINY)
    w = llama_ref.make_weights(cfg, 42)
    toks = np.random.default_rng([2, 0, 0]).integers(0, 2 ** 32, size=256, dtype=np.uint32)
    a = llama_ref.llama_forward(cfg, w, toks, [9642, 2822], round_bf16=True)[0]
    b = llama_ref.llama_forward(cfg, w, toks, [9642, 2822], round_bf16=False)[0]
    assert np.abs(a - b).max() < 5e-2

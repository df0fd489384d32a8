"""End-to-end PrefillOnly forward on the GPU vs the CPU oracle (oracle/llama_ref.py).

Bar (north star): allowed-token argmax bit-exact, logits within a stated BF16 tolerance:
    |logit_gpu - logit_oracle| <= LOGIT_ATOL + LOGIT_RTOL * |logit_oracle|
The argmax must equal the oracle's in every case. The cases use fixed seeds; each test prints the oracle's top-2
margin, and a case whose margin fell inside the tolerance band would be a failure to decide, not a pass.
"""

import numpy as np
import pytest

from oracle import llama_ref
from paper_2505_07203_b200.config import ModelConfig, TINY
from paper_2505_07203_b200.engine import CapacityError, Engine

pytestmark = pytest.mark.gpu

LOGIT_ATOL = 1e-2  # measured max |error|: 9e-4 (tiny) .. 7.5e-3 (round 1, all cases)
LOGIT_RTOL = 5e-3
YES_NO = [9642, 2822]  # build-chosen "Yes"/"No" ids (Llama-3 tokenizer ids), valid in every preset vocab

SMALL = ModelConfig("small", 2, 1024, 8, 2, 128, 2816, 4096)
# Qwen2-style: odd GQA group (5), q/k/v bias, plain RoPE theta 1e6, eps 1e-6 (Qwen-2.5-32B family at tiny size)
TINY_QWEN = ModelConfig("tiny-qwen", 2, 1280, 10, 2, 128, 1024, 32000, rms_eps=1e-6, rope_theta=1_000_000.0,
                        rope_scaling=0, qkv_bias=True)


def tokens_for(seed: int, n: int) -> np.ndarray:
    # same stream construction as the reference workloads (ps/workload.py:113-115)
    return np.random.default_rng([seed, 0, 0]).integers(0, 2 ** 32, size=n, dtype=np.uint32)


_weights = {}


def oracle_weights(model, seed):
    key = (model.name, seed)
    if key not in _weights:
        _weights[key] = llama_ref.make_weights(llama_ref.Cfg.from_model(model), seed)
    return _weights[key]


def check_against_oracle(model, res, toks, allowed, seed):
    cfg = llama_ref.Cfg.from_model(model)
    logits, probs, am = llama_ref.llama_forward(cfg, oracle_weights(model, seed), toks, allowed)
    err = np.abs(res.logits - logits)
    tol = LOGIT_ATOL + LOGIT_RTOL * np.abs(logits)
    print(f"{model.name}: n={len(toks)} logits gpu={res.logits} oracle={logits} max_err={err.max():.3e}")
    assert (err <= tol).all(), (res.logits, logits)
    srt = np.sort(logits)[::-1]
    margin = srt[0] - srt[1] if len(srt) > 1 else np.inf
    print(f"  oracle top-2 margin {margin:.3e} (tolerance band {tol.max():.3e})")
    assert res.index == am, f"argmax {res.index} != oracle {am} (margin {margin:.3e})"
    assert np.allclose(res.probs.sum(), 1.0, atol=1e-5)


@pytest.fixture(scope="module")
def tiny_engine():
    with Engine(TINY, seed=42, max_tokens=4096, chunk=1024, pool_blocks=512) as e:
        yield e


def test_tiny_2k_request_matches_oracle(tiny_engine):
    toks = tokens_for(0, 2048)
    res = tiny_engine.prefill(toks, YES_NO)
    check_against_oracle(TINY, res, toks, YES_NO, 42)
    assert res.token in YES_NO and res.service_s > 0


@pytest.mark.parametrize("n", [1, 17, 130, 1000])
def test_tiny_ragged_lengths(tiny_engine, n):
    toks = tokens_for(n, n)
    res = tiny_engine.prefill(toks, YES_NO)
    check_against_oracle(TINY, res, toks, YES_NO, 42)


def test_tiny_many_allowed_ids(tiny_engine):
    toks = tokens_for(3, 700)
    allowed = list(range(0, 32000, 97))
    res = tiny_engine.prefill(toks, allowed)
    check_against_oracle(TINY, res, toks, allowed, 42)


def test_tiny_whole_vocab_allowed(tiny_engine):
    # the LM head spreads a long allowed list over many CTAs (one per SM at most) and the last one runs the softmax
    toks = tokens_for(5, 300)
    allowed = list(range(32000))
    res = tiny_engine.prefill(toks, allowed)
    check_against_oracle(TINY, res, toks, allowed, 42)
    again = tiny_engine.prefill(toks, allowed)
    assert np.array_equal(res.logits, again.logits) and res.index == again.index


def test_small_gqa_chunked_mlp():
    toks = tokens_for(9, 1500)
    with Engine(SMALL, seed=7, max_tokens=2048, chunk=512, pool_blocks=64) as e:
        res = e.prefill(toks, [5, 11, 4095])
    check_against_oracle(SMALL, res, toks, [5, 11, 4095], 7)


def test_qwen_style_odd_group_and_bias():
    toks = tokens_for(17, 1300)
    with Engine(TINY_QWEN, seed=5, max_tokens=2048, chunk=512, pool_blocks=128) as e:
        res = e.prefill(toks, YES_NO)
        check_against_oracle(TINY_QWEN, res, toks, YES_NO, 5)
        # prefix hit through the pool on the query-block-pair attention path
        slots = list(range(1300 // 16))
        e.prefill(toks, YES_NO, 0, slots)
        warm = e.prefill(toks, YES_NO, 1024, slots)
        check_against_oracle(TINY_QWEN, warm, toks, YES_NO, 5)


def test_chunk_size_does_not_change_result():
    toks = tokens_for(4, 1300)
    outs = {}
    for chunk in (128, 512, 1024, 8192):
        with Engine(TINY, seed=42, max_tokens=2048, chunk=chunk, pool_blocks=8) as e:
            outs[chunk] = e.prefill(toks, YES_NO)
    # per-row ops: chunking must be bit-exact (ps/numerics.py docstring: chunking cannot change a result). Chunks of
    # >= 512 rows run the fused MLP launch (row pieces of chunk / 2 in the L2 ring): identical bits for every size.
    assert all(np.array_equal(outs[512].logits, outs[c].logits) for c in (1024, 8192))
    # 128-row chunks run per-chunk short-M GEMM launches (split-K over the weight: another summation order)
    check_against_oracle(TINY, outs[128], toks, YES_NO, 42)
    assert outs[128].index == outs[512].index


def test_prefix_pool_reuse_matches_oracle(tiny_engine):
    """K/V served from the prefix pool (cached rows only act as keys) gives the oracle's answer.

    Short-query requests run split-KV attention (different summation order than the cold forward), so
    warm and cold forwards agree within the stated tolerance rather than bit for bit.
    """
    bt = 16
    base = tokens_for(11, 1024)
    slots_a = list(range(100, 164))  # request A: cold, admit all 64 blocks into slots 100..163
    tiny_engine.prefill(base, YES_NO, n_cached=0, pool_block_ids=slots_a)
    b = np.concatenate([base[:640], tokens_for(12, 500)])  # request B shares A's first 640 tokens
    n_cached = 640
    ids = slots_a[: n_cached // bt] + [-1] * (len(b) // bt - n_cached // bt)
    warm = tiny_engine.prefill(b, YES_NO, n_cached=n_cached, pool_block_ids=ids)
    assert warm.n_cached == 640
    check_against_oracle(TINY, warm, b, YES_NO, 42)
    cold = tiny_engine.prefill(b, YES_NO)
    assert np.abs(warm.logits - cold.logits).max() <= LOGIT_ATOL
    # fully cached request: only the last token is recomputed
    full = tiny_engine.prefill(base, YES_NO, n_cached=1024, pool_block_ids=slots_a)
    check_against_oracle(TINY, full, base, YES_NO, 42)


def test_admission_writes_pool_then_long_hit(tiny_engine):
    """Blocks admitted by one request (K/V written during its forward) serve a later, longer request."""
    base = tokens_for(21, 3000)
    slots = list(range(200, 200 + 3000 // 16))
    tiny_engine.prefill(base[:2048], YES_NO, 0, slots[:128])
    res = tiny_engine.prefill(base, YES_NO, 2048, slots[:128] + [-1] * (3000 // 16 - 128))
    check_against_oracle(TINY, res, base, YES_NO, 42)


def test_last_row_only_equals_full_last_layer():
    toks = tokens_for(31, 1700)
    res = {}
    for flag in (True, False):
        with Engine(TINY, seed=42, max_tokens=2048, chunk=512, pool_blocks=8, last_row_only=flag) as e:
            res[flag] = e.prefill(toks, YES_NO)
            check_against_oracle(TINY, res[flag], toks, YES_NO, 42)
    assert np.abs(res[True].logits - res[False].logits).max() <= LOGIT_ATOL


def test_capacity_error(tiny_engine):
    with pytest.raises(CapacityError):
        tiny_engine.prefill(tokens_for(0, 4097), YES_NO)


def test_arena_matches_geometry_model():
    """The engine's allocation is the hybrid-mode peak the geometry module predicts (the profile run)."""
    from paper_2505_07203_b200 import geometry
    from paper_2505_07203_b200.config import LLAMA_3_1_8B

    from paper_2505_07203_b200.config import TINY_FP8

    for model, T, chunk in ((TINY, 4096, 1024), (SMALL, 2048, 512), (LLAMA_3_1_8B, 24_000, 8192),
                            (TINY_FP8, 4096, 1024)):
        with Engine(model, seed=0, max_tokens=T, chunk=chunk, pool_blocks=4) as e:
            assert e.arena_bytes == geometry.arena_bytes(model, T, chunk)
            norms_fp32_extra = (2 * model.num_layers + 1) * model.hidden * 2  # norms held as fp32 on device
            assert e.weight_bytes == model.weight_bytes + norms_fp32_extra
            assert e.block_bytes == model.kv_bytes_per_token[1] * 16


@pytest.mark.parametrize("n_cached", [16, 656, 1008])
def test_pool_direct_straddling_tiles_match_oracle(tiny_engine, n_cached):
    """Cached K/V read by attention straight from the pool: a cached prefix that ends inside a 128-key tile mixes
    pool blocks and freshly computed qkv rows in one tile (16-key boxes from each source)."""
    bt = 16
    base = tokens_for(21, 1200)
    slots = list(range(200, 200 + len(base) // bt))
    tiny_engine.prefill(base, YES_NO, n_cached=0, pool_block_ids=slots)
    req = np.concatenate([base[:n_cached], tokens_for(22, 300)])
    ids = slots[: n_cached // bt] + [-1] * (len(req) // bt - n_cached // bt)
    warm = tiny_engine.prefill(req, YES_NO, n_cached=n_cached, pool_block_ids=ids)
    assert warm.n_cached == n_cached
    check_against_oracle(TINY, warm, req, YES_NO, 42)


def test_pool_slot_layouts_read_the_same_kv(tiny_engine):
    """Pool-direct attention loads a whole cached 128-key tile whose eight blocks sit in consecutive slots as two
    4-D boxes ([slot][layer][16][kv_dim]) and any other tile block by block. The same request cached under
    consecutive, scattered and mixed slot layouts must give bit-identical hits, and match the oracle."""
    bt = 16
    base = tokens_for(23, 2000)
    nb = len(base) // bt  # 125 blocks: 15 whole tiles + a partial one
    n_cached = 1920
    rng = np.random.default_rng(5)
    pool = np.arange(260, 512)
    mixed = []
    for t in range((nb + 7) // 8):  # even tiles one consecutive run at a random start, odd tiles scattered
        k = min(8, nb - 8 * t)
        if t % 2 == 0:
            start = 260 + 16 * t + int(rng.integers(0, 8))
            mixed += list(range(start, start + k))
        else:
            mixed += [int(x) for x in rng.choice(pool[(pool >= 260 + 16 * t) & (pool < 260 + 16 * t + 16)], k,
                                                 replace=False)]
    layouts = {
        "consecutive": list(range(300, 300 + nb)),
        "scattered": [int(x) for x in rng.permutation(np.arange(300, 300 + nb))],
        "mixed": mixed,
    }
    hits = {}
    for name, slots in layouts.items():
        assert len(set(slots)) == nb and all(0 <= x < 512 for x in slots)
        tiny_engine.prefill(base, YES_NO, n_cached=0, pool_block_ids=slots)
        ids = slots[: n_cached // bt] + [-1] * (nb - n_cached // bt)
        hits[name] = tiny_engine.prefill(base, YES_NO, n_cached=n_cached, pool_block_ids=ids)
        assert hits[name].n_cached == n_cached
    for name in ("scattered", "mixed"):
        assert np.array_equal(hits[name].logits, hits["consecutive"].logits), name
    check_against_oracle(TINY, hits["mixed"], base, YES_NO, 42)


@pytest.mark.parametrize("model", [TINY, SMALL], ids=["tiny", "small-splitk"])
def test_short_suffix_admission_feeds_later_hits(model):
    """A prefix hit with a short miss suffix admits its suffix blocks from the QKV epilogue (the pair GEMM for the
    tiny model, the split-K reduce for `small`); a later request whose cached prefix covers those blocks must match
    the oracle."""
    slots = list(range(300, 300 + 80))
    allowed = [a % model.vocab for a in YES_NO]
    with Engine(model, seed=42, max_tokens=2048, chunk=1024, pool_blocks=512) as eng:
        a_toks = tokens_for(31, 640)
        eng.prefill(a_toks, allowed, n_cached=0, pool_block_ids=slots[:40])       # A: admit 40 blocks
        b_toks = np.concatenate([a_toks, tokens_for(32, 160)])                     # B: hit + 160-token suffix
        b = eng.prefill(b_toks, allowed, n_cached=640, pool_block_ids=slots[:50])  # admits blocks 40..49
        check_against_oracle(model, b, b_toks, allowed, 42)
        c_toks = np.concatenate([b_toks, tokens_for(33, 48)])                      # C: cached through B's suffix
        c = eng.prefill(c_toks, allowed, n_cached=800, pool_block_ids=slots[:50] + [-1] * 3)
        assert c.n_cached == 800
        check_against_oracle(model, c, c_toks, allowed, 42)


def test_request_validation_errors(tiny_engine):
    """Bad requests fail loudly with the reference taxonomy and leave the engine usable."""
    from paper_2505_07203_b200._lib import PrefillOnlyError

    toks = tokens_for(30, 256)
    slots = list(range(300, 316))
    bad = [
        dict(tokens=toks[:0], allowed=YES_NO),                                    # empty request
        dict(tokens=toks, allowed=[]),                                           # empty allowed list
        dict(tokens=toks, allowed=[32_000]),                                     # id past the vocab
        dict(tokens=toks, allowed=[-1]),
        dict(tokens=toks, allowed=YES_NO, n_cached=8, pool_block_ids=slots),     # not block aligned
        dict(tokens=toks, allowed=YES_NO, n_cached=272, pool_block_ids=slots),   # n_cached > n
        dict(tokens=toks, allowed=YES_NO, n_cached=32, pool_block_ids=[1]),      # cached blocks without slots
        dict(tokens=toks, allowed=YES_NO, n_cached=0, pool_block_ids=[10 ** 6]),  # admit slot out of range
        dict(tokens=toks, allowed=YES_NO, n_cached=0, pool_block_ids=[7, 7]),    # two admitted blocks, one slot
        dict(tokens=toks, allowed=YES_NO, n_cached=16, pool_block_ids=[7, 7]),   # admission over a cached block
    ]
    for kw in bad:
        with pytest.raises((PrefillOnlyError, ValueError)):
            tiny_engine.prefill(**kw)
    ok = tiny_engine.prefill(toks, [5, 5, 9])  # duplicate allowed ids are legal: equal logits, first max wins
    assert ok.logits[0] == ok.logits[1] and ok.index != 1
    check_against_oracle(TINY, tiny_engine.prefill(toks, YES_NO), toks, YES_NO, 42)


def test_back_to_back_async_hits_use_their_own_slot_tables(tiny_engine):
    """po_prefill_device returns before its forward runs. Two prefix hits issued back to back behind a long cold
    forward, with different cached slot tables, must each read their own pool slots (the staging ring keeps the
    first call's block table alive until its forward has consumed it)."""
    import torch

    bt = 16
    a, b = tokens_for(41, 1200), tokens_for(42, 1200)
    slots_a = list(range(0, 75))
    slots_b = list(range(100, 175))
    tiny_engine.prefill(a, YES_NO, 0, slots_a)
    tiny_engine.prefill(b, YES_NO, 0, slots_b)
    dev = torch.device("cuda", 0)
    stream = tiny_engine.stream
    busy = torch.from_numpy(tokens_for(43, 4000).view(np.int32)).to(dev)
    d_a = torch.from_numpy(a.view(np.int32)).to(dev)
    d_b = torch.from_numpy(b.view(np.int32)).to(dev)
    alw = torch.tensor(YES_NO, dtype=torch.int32, device=dev)
    outs = [(torch.empty(2, device=dev), torch.empty(2, device=dev), torch.empty(1, dtype=torch.int32, device=dev))
            for _ in range(3)]
    torch.cuda.synchronize()
    nc = 1024
    for (lg, pr, am), d_tok, slots, n_c, n in ((outs[0], busy, [], 0, 4000), (outs[1], d_a, slots_a, nc, 1200),
                                               (outs[2], d_b, slots_b, nc, 1200)):
        tiny_engine.prefill_device(d_tok.data_ptr(), n, alw.data_ptr(), 2, lg.data_ptr(), pr.data_ptr(),
                                   am.data_ptr(), n_cached=n_c, pool_block_ids=slots[: n_c // bt])
    torch.cuda.synchronize()
    for (lg, pr, am), toks in ((outs[1], a), (outs[2], b)):
        res = type("R", (), {})()
        res.logits, res.probs, res.index = lg.cpu().numpy(), pr.cpu().numpy(), int(am.item())
        check_against_oracle(TINY, res, toks, YES_NO, 42)


@pytest.fixture(scope="module")
def small_engine():
    with Engine(SMALL, seed=7, max_tokens=2048, chunk=1024, pool_blocks=256) as e:
        yield e


@pytest.mark.parametrize("n", [1, 100, 128, 129, 200, 256])
def test_streaming_kernel_short_requests_match_oracle(small_engine, n):
    """Requests of <= 256 miss rows run their layer GEMMs as phases of the persistent weight-streaming kernel
    (stream.cu: stream-K split of every weight matrix over the SM pairs, in-kernel fix-up, grid barriers between the
    O / gate-up / down / next-QKV phases). M = 1 leaves the second CTA of each pair without rows; 129 crosses it."""
    toks = tokens_for(50 + n, n)
    res = small_engine.prefill(toks, [5, 11, 4095])
    check_against_oracle(SMALL, res, toks, [5, 11, 4095], 7)


def test_streaming_kernel_hit_suffixes_match_oracle(small_engine):
    """Prefix hits with 160- and 256-row suffixes (the serving hot path) and admission from the streamed QKV phase."""
    base = tokens_for(60, 1600)
    slots = list(range(0, 100))
    small_engine.prefill(base[:1344], [5, 11, 4095], 0, slots[:84])
    for n_cached, n in ((1344, 1504), (1344, 1600)):
        toks = base[:n]
        res = small_engine.prefill(toks, [5, 11, 4095], n_cached, slots[: n // 16])
        check_against_oracle(SMALL, res, toks, [5, 11, 4095], 7)
    # blocks 84..99 were admitted by the streamed QKV epilogue of the second hit: serve them as cached keys
    res = small_engine.prefill(base, [5, 11, 4095], 1584, slots)
    check_against_oracle(SMALL, res, base, [5, 11, 4095], 7)

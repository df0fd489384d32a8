"""Product prefix-pool manager (paper_2505_07203_b200/cache.py) vs the reference fixtures and the oracle.

Covers the reference's own cache tests (pkg/tests/test_cache.py): partial-block drop, block-boundary
match, read-only probe, suffix discard at capacity, LRU touch, self-eviction protection, evict_to,
randomised invariants — plus the B200 additions: pool slots and two-phase admission.
"""

import numpy as np
import pytest

from golden_util import golden
from oracle import sched_ref
from paper_2505_07203_b200.cache import (CacheConfig, CacheError, EvictionShortfall, PrefixCache,
                                         block_chain)


def toks(*ranges):
    return np.concatenate([np.arange(a, b, dtype=np.uint32) for a, b in ranges])


def make(cap, bt=16):
    return PrefixCache(CacheConfig(capacity_tokens=cap, block_tokens=bt))


def test_block_chain_matches_reference_fixtures():
    for c in golden()["block_chains"]:
        t = np.random.default_rng([c["seed"], 77]).integers(0, 2 ** 32, size=c["n"], dtype=np.uint32)
        assert [d.hex() for d in block_chain(t, c["bt"])] == c["chain"]


def test_block_chain_base_extension():
    t = toks((0, 100))
    base = block_chain(t[:48], 16)
    assert block_chain(t, 16, base=base) == block_chain(t, 16)
    with pytest.raises(CacheError):
        block_chain(t[:16], 16, base=base)


def test_golden_op_sequence_and_slots():
    g = golden()["cache_ops"]
    chains = [block_chain(np.array(s, dtype=np.uint32), g["bt"]) for s in g["seqs"]]
    c = make(g["capacity_tokens"], g["bt"])
    for op in g["ops"]:
        if op["op"] == "insert":
            assert c.insert_chain(chains[op["seq"]], op["now"]) == op["out"]
        elif op["op"] == "match":
            assert c.match_chain(chains[op["seq"]]) == op["out"]
        else:
            if op["out"] >= 0:
                assert c.evict_to(op["need"], protect=chains[op["seq"]]) == op["out"]
            else:
                with pytest.raises(EvictionShortfall):
                    c.evict_to(op["need"], protect=chains[op["seq"]])
        assert c.used_tokens == op["used"]
        c.check_invariants()
    assert sorted(d.hex() for d in c._blocks) == g["final_resident"]


def test_partial_block_ignored_and_boundary_match():
    c = make(4096)
    assert c.insert(toks((0, 40)), now=0.0) == 32
    assert c.match(toks((0, 40))) == 32
    assert c.match(toks((0, 32))) == 32
    assert c.match(toks((0, 31))) == 16
    assert c.match(toks((1, 40))) == 0


def test_probe_is_read_only():
    c = make(4096)
    c.insert(toks((0, 64)), now=0.0)
    v = c.version
    for _ in range(3):
        c.match(toks((0, 64)))
    assert c.version == v


def test_suffix_discard_at_capacity():
    c = make(64)
    assert c.insert(toks((0, 160)), now=0.0) == 64
    assert c.used_tokens == 64
    c.check_invariants()


def test_lru_touch_and_self_protection():
    c = make(64)
    c.insert(toks((0, 32)), now=0.0)
    c.insert(toks((1000, 1032)), now=1.0)
    c.insert(toks((0, 32)), now=2.0)  # touch the first sequence
    c.insert(toks((2000, 2032)), now=3.0)  # evicts the LRU leaf chain (1000..)
    assert c.match(toks((0, 32))) == 32
    assert c.match(toks((1000, 1032))) == 0
    # a long insertion never evicts its own path
    assert c.insert(toks((5000, 5160)), now=4.0) == 64
    c.check_invariants()


def test_random_ops_vs_oracle():
    rng = np.random.default_rng(7)
    bases = [rng.integers(0, 2 ** 32, size=16 * 30, dtype=np.uint32) for _ in range(8)]
    seqs = [np.concatenate([bases[int(rng.integers(0, 8))][: int(rng.integers(1, 31)) * 16],
                            rng.integers(0, 2 ** 32, size=int(rng.integers(0, 40)), dtype=np.uint32)])
            for _ in range(60)]
    chains = [block_chain(s, 16) for s in seqs]
    for cap_blocks in (1, 7, 40, 200):
        mine, ref = make(16 * cap_blocks), sched_ref.PrefixCache(16 * cap_blocks)
        now = 0.0
        for _ in range(1500):
            now += float(rng.integers(0, 2))
            k = int(rng.integers(0, len(chains)))
            r = rng.random()
            if r < 0.5:
                assert mine.insert_chain(chains[k], now) == ref.insert_chain(chains[k], now)
            elif r < 0.9:
                assert mine.match_chain(chains[k]) == ref.match_chain(chains[k])
            else:
                need = int(rng.integers(0, cap_blocks + 1)) * 16
                try:
                    a = mine.evict_to(need, chains[k])
                except EvictionShortfall:
                    a = None
                try:
                    b = ref.evict_to(need, chains[k])
                except ValueError:
                    b = None
                assert a == b
            assert set(mine._blocks) == set(ref.blocks)
        mine.check_invariants()


def test_two_phase_admission_equals_one_shot_and_committed_view():
    rng = np.random.default_rng(3)
    seqs = [rng.integers(0, 2 ** 32, size=int(rng.integers(16, 400)), dtype=np.uint32) for _ in range(30)]
    seqs += [np.concatenate([seqs[i][: 16 * (len(seqs[i]) // 32)], seqs[i + 1]]) for i in range(10)]
    chains = [block_chain(s, 16) for s in seqs]
    a, b = make(16 * 50), make(16 * 50)
    t = 0.0
    for k in rng.integers(0, len(chains), size=300):
        t += 1.0
        ch = chains[int(k)]
        before = {d: a.match_chain(chains[j]) for j, d in enumerate(range(len(chains)))}
        adm = b.begin_insert(ch, t)
        # while in flight, the committed view is the pre-insert state
        for j, other in enumerate(chains):
            assert b.match_chain(other, committed=True) == before[j]
        # admitted blocks are exactly the newly stored ones, slots distinct and in range
        slots = [s for _, s in adm.admit]
        assert len(set(slots)) == len(slots) and all(0 <= s < 50 for s in slots)
        b.commit(adm, t + 0.5)
        a.insert_chain(ch, t + 0.5)
        assert set(a._blocks) == set(b._blocks)
        assert all(a._blocks[d].last_use == b._blocks[d].last_use for d in a._blocks)
        b.check_invariants()
    # pool_block_ids: cached slots first, then admissions, -1 for discarded blocks
    c = make(16 * 4)
    ch = block_chain(np.arange(16 * 6, dtype=np.uint32), 16)
    adm = c.begin_insert(ch, 0.0)
    ids = adm.pool_block_ids(0, [])
    assert len(ids) == 6 and ids[4:] == [-1, -1] and sorted(ids[:4]) == [0, 1, 2, 3]
    c.commit(adm, 1.0)
    n = c.match_chain(ch)
    assert n == 64 and c.slots(ch, 4) == ids[:4]


def test_abort_drops_unwritten_blocks():
    c = make(16 * 8)
    adm = c.begin_insert(block_chain(np.arange(64, dtype=np.uint32), 16), 0.0)
    c.abort(adm)
    assert c.resident_blocks == 0
    c.check_invariants()


def test_config_validation():
    with pytest.raises(CacheError):
        CacheConfig(capacity_tokens=-1)
    with pytest.raises(CacheError):
        CacheConfig(capacity_tokens=16, block_tokens=0)
    with pytest.raises(CacheError):
        make(32).evict_to(64)


def test_readmitted_blocks_take_ascending_consecutive_slots():
    """Slots come from a min-heap and are handed out after an insertion's evictions: blocks admitted in place of a
    chain evicted leaf by leaf (last block first) get ascending consecutive slots, so pool-direct attention can load
    whole 8-block tiles as one box."""
    c = make(64 * 16)
    a = toks((0, 40 * 16))
    b = toks((100000, 100000 + 40 * 16))
    c.insert(a, now=0.0)
    ca = block_chain(a, 16)
    assert c.slots(ca, 40) == list(range(40))
    c.insert(b, now=1.0)  # needs 16 of a's blocks: its tail 24..39 is evicted (last block first) while b is planned
    cb = block_chain(b, 16)
    sb = c.slots(cb, 40)
    assert sb == list(range(24, 64))  # slots are handed out after the evictions, lowest first, in chain order
    for t in range(5):
        run = sb[8 * t: 8 * t + 8]
        assert run == list(range(run[0], run[0] + 8))
    c.check_invariants()

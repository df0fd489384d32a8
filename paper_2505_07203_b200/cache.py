"""Prefix-KV pool manager: block-digest trie, LRU leaf eviction, suffix discard, pool slots.

Policy semantics follow the reference PrefixCache (ps/cache.py:92-211):
  * blocks of `block_tokens` tokens keyed by chained blake2b-128 digests (ps/cache.py:39-62);
  * lookups binary-search the chain using prefix closure (ps/cache.py:119-130), read-only (Q5);
  * insertion touches resident path blocks, admits new blocks while capacity allows, evicting the LRU
    unprotected leaf (min (last_use, ins_order), Q8); it stops at the first block it cannot place and drops
    the suffix (Q7, suffix discard).
What is new here is the binding to GPU memory: every resident block owns a slot of the engine's prefix pool
([slot][layer][16][kv] bf16, csrc/engine.cu), and admission is two-phase because the K/V of an admitted
block is written *during* its request's forward while the reference admits at *completion*
(ps/sim.py:255-257):
  begin_insert(chain, now_start) -> Admission   decisions + slots, applied tentatively;
  commit(admission, now_done)                   re-stamps the path with the completion time.
Between the two, `match_chain(..., committed=True)` answers from the pre-insert state, so an arrival-time
probe (static SRJF, Q3) sees exactly what the reference sees. Victim search uses a lazy min-heap instead of
the reference's O(#leaves) scan; the chosen victims are identical (tests/test_cache_parity.py).
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass, field
from hashlib import blake2b
from typing import Sequence

import numpy as np

DIGEST_SIZE = 16


class CacheError(ValueError):
    """Invalid cache configuration or operation."""


class EvictionShortfall(CacheError):
    def __init__(self, needed_tokens: int, freed_tokens: int):
        self.needed_tokens = needed_tokens
        self.freed_tokens = freed_tokens
        super().__init__(f"needed {needed_tokens} tokens but only {freed_tokens} were evictable")


def block_chain(tokens, block_tokens: int, base: Sequence[bytes] = ()) -> list[bytes]:
    """Digest chain of the full blocks: d_i = blake2b(d_{i-1} || uint32-LE tokens of block i, 16 B)."""
    if block_tokens < 1:
        raise CacheError("block_tokens must be >= 1")
    arr = np.ascontiguousarray(tokens, dtype="<u4")
    nb = arr.shape[0] // block_tokens
    out = list(base)
    if len(out) > nb:
        raise CacheError("base chain longer than the sequence's block count")
    raw = arr[: nb * block_tokens].tobytes()
    stride = 4 * block_tokens
    prev = out[-1] if out else b""
    for i in range(len(out), nb):
        prev = blake2b(prev + raw[i * stride:(i + 1) * stride], digest_size=DIGEST_SIZE).digest()
        out.append(prev)
    return out


@dataclass(frozen=True)
class CacheConfig:
    capacity_tokens: int
    block_tokens: int = 16

    def __post_init__(self):
        if self.block_tokens < 1:
            raise CacheError("block_tokens must be >= 1")
        if self.capacity_tokens < 0:
            raise CacheError("capacity_tokens must be >= 0")

    @property
    def capacity_blocks(self) -> int:
        return self.capacity_tokens // self.block_tokens


class _Node:
    __slots__ = ("parent", "depth", "children", "last_use", "ins_order", "slot")

    def __init__(self, parent, depth, last_use, ins_order, slot):
        self.parent = parent
        self.depth = depth
        self.children = 0
        self.last_use = last_use
        self.ins_order = ins_order
        self.slot = slot


@dataclass
class Admission:
    """Decisions of one insertion: what the forward must write and what it may overwrite."""

    chain: list
    stored_blocks: int  # resident prefix blocks of this chain after insertion
    admit: list = field(default_factory=list)  # (block index, slot) of newly admitted blocks
    evicted: dict = field(default_factory=dict)  # digest -> _Node removed to make room
    touched: list = field(default_factory=list)  # digests whose last_use the insertion stamps
    new_set: set = field(default_factory=set)  # digests of newly admitted blocks
    committed: bool = False

    def pool_block_ids(self, n_cached_blocks: int, slots_of_cached: Sequence[int]) -> list[int]:
        """po_prefill's pool_block_ids: cached slots, then admission slots (-1 = discarded)."""
        ids = list(slots_of_cached[:n_cached_blocks])
        admit = dict(self.admit)
        ids += [admit.get(b, -1) for b in range(n_cached_blocks, len(self.chain))]
        return ids


class PrefixCache:
    """LRU prefix cache over block digest chains, bound to prefix-pool slots."""

    def __init__(self, config: CacheConfig):
        self.config = config
        self._blocks: dict[bytes, _Node] = {}
        self._leaf_heap: list = []  # (last_use, ins_order, digest), lazily invalidated
        self._ins_counter = 0
        # free pool slots as a min-heap: admissions take the lowest free slots, so a request's new blocks (and the
        # blocks of a chain evicted leaf by leaf and re-admitted) land in ascending consecutive slots, which
        # pool-direct attention loads as whole-tile boxes (csrc/attention.cu)
        self._free_slots = list(range(config.capacity_blocks))
        self._pending: Admission | None = None
        self.version = 0

    # ------------------------------------------------------------------ inspection
    @property
    def used_tokens(self) -> int:
        return len(self._blocks) * self.config.block_tokens

    @property
    def resident_blocks(self) -> int:
        return len(self._blocks)

    def _resident(self, d: bytes, committed: bool) -> bool:
        if committed and self._pending is not None:
            p = self._pending
            if d in p.evicted:
                return True
            if d in self._blocks and d in p.new_set:
                return False
        return d in self._blocks

    def match(self, tokens, committed: bool = False) -> int:
        return self.match_chain(block_chain(tokens, self.config.block_tokens), committed)

    def match_chain(self, chain: Sequence[bytes], committed: bool = False) -> int:
        """Tokens of the longest resident block-aligned prefix (read-only)."""
        if not chain:
            return 0
        res = self._resident if committed and self._pending is not None else None
        present = (lambda d: res(d, True)) if res else self._blocks.__contains__
        if not present(chain[0]):
            return 0
        lo, hi = 1, len(chain)
        while lo < hi:
            mid = (lo + hi + 1) >> 1
            if present(chain[mid - 1]):
                lo = mid
            else:
                hi = mid - 1
        return lo * self.config.block_tokens

    def slots(self, chain: Sequence[bytes], n_blocks: int) -> list[int]:
        return [self._blocks[d].slot for d in chain[:n_blocks]]

    # ------------------------------------------------------------------ mutation
    def insert(self, tokens, now: float) -> int:
        return self.insert_chain(block_chain(tokens, self.config.block_tokens), now)

    def insert_chain(self, chain: Sequence[bytes], now: float) -> int:
        """Reference-equivalent one-shot insertion (ps/cache.py:143-159)."""
        adm = self.begin_insert(chain, now)
        self.commit(adm, now)
        return adm.stored_blocks * self.config.block_tokens

    def begin_insert(self, chain: Sequence[bytes], now: float) -> Admission:
        """Plan an insertion (ps/cache.py:143-159): the resident prefix is found by the prefix-closed binary search,
        then the suffix blocks are admitted (evicting LRU leaves off the path) until one cannot be.

        Last-use stamps are kept lazily: an insertion stamps only its deepest stored block, and a block that loses
        its last child takes the child's stamp if it is later (`_remove`). Only leaves are eviction candidates, and
        a leaf's lazy stamp equals the reference's eager one (the latest insertion whose path ran through it), so
        victims and tie-breaks are identical while an insertion costs O(new blocks) instead of O(chain)."""
        if self._pending is not None:
            raise CacheError("an insertion is already in flight on this instance")
        self.version += 1
        self._maybe_compact()
        chain = list(chain)
        n_res = self.match_chain(chain) // self.config.block_tokens
        adm = Admission(chain=chain, stored_blocks=n_res)
        cap = self.config.capacity_blocks
        path = None
        for i in range(n_res, len(chain)):
            d = chain[i]
            if len(self._blocks) >= cap:
                if path is None:
                    path = set(chain)
                victim = self._evict_one(path)
                if victim is None:
                    break  # this block and the whole suffix are discarded
                adm.evicted[victim[0]] = victim[1]
            self._add_block(d, chain[i - 1] if i > 0 else None, now, take_slot=False)
            adm.admit.append((i, -1))
            adm.new_set.add(d)
            adm.stored_blocks = i + 1
        # slots after the evictions: the admitted blocks take the lowest free slots in chain order (ascending runs)
        for j, (i, _) in enumerate(adm.admit):
            slot = heapq.heappop(self._free_slots)
            self._blocks[chain[i]].slot = slot
            adm.admit[j] = (i, slot)
        if adm.stored_blocks:
            d = chain[adm.stored_blocks - 1]
            self._stamp(d, self._blocks[d], now)
            adm.touched.append(d)
        self._pending = adm
        return adm

    def commit(self, adm: Admission, now: float):
        """Finish an insertion: stamp the path with the completion time (the reference inserts at completion)."""
        if adm is not self._pending:
            raise CacheError("commit of an admission that is not in flight")
        # the deepest stored block and the newly admitted ones (so a two-phase insertion leaves the same stamps as a
        # one-shot insertion at the completion time)
        for d in adm.touched + [adm.chain[b] for b, _ in adm.admit]:
            node = self._blocks.get(d)
            if node is not None and node.last_use != now:
                self._stamp(d, node, now)
        adm.committed = True
        self._pending = None

    def abort(self, adm: Admission):
        """Drop an in-flight admission whose forward failed: its new blocks never received K/V."""
        if adm is not self._pending:
            raise CacheError("abort of an admission that is not in flight")
        for b, _ in reversed(adm.admit):
            d = adm.chain[b]
            if d in self._blocks and self._blocks[d].children == 0:
                self._remove(d)
        self._pending = None
        self.version += 1

    def evict_to(self, needed_tokens: int, protect: Sequence[bytes] = ()) -> int:
        if needed_tokens > self.config.capacity_tokens:
            raise CacheError("cannot free more than the cache capacity")
        protected = set(protect)
        freed = 0
        while self.config.capacity_tokens - self.used_tokens < needed_tokens:
            if self._evict_one(protected) is None:
                raise EvictionShortfall(needed_tokens, freed)
            freed += self.config.block_tokens
        if freed:
            self.version += 1
        return freed

    # ------------------------------------------------------------------ internals
    def _maybe_compact(self):
        if len(self._leaf_heap) > 4 * len(self._blocks) + 1024:
            self._leaf_heap = [(n.last_use, n.ins_order, d) for d, n in self._blocks.items() if n.children == 0]
            heapq.heapify(self._leaf_heap)

    def _stamp(self, d: bytes, node: _Node, now: float):
        node.last_use = now
        if node.children == 0:
            heapq.heappush(self._leaf_heap, (node.last_use, node.ins_order, d))

    def _add_block(self, d: bytes, parent, now: float, take_slot: bool = True) -> int:
        self._ins_counter += 1
        if not self._free_slots:
            raise CacheError("prefix pool has no free slot")  # cannot happen: capacity checked first
        slot = heapq.heappop(self._free_slots) if take_slot else -1
        depth = 1 if parent is None else self._blocks[parent].depth + 1
        node = _Node(parent, depth, now, self._ins_counter, slot)
        self._blocks[d] = node
        heapq.heappush(self._leaf_heap, (now, node.ins_order, d))
        if parent is not None:
            self._blocks[parent].children += 1
        return slot

    def _valid_leaf(self, entry) -> bool:
        node = self._blocks.get(entry[2])
        return node is not None and node.children == 0 and node.last_use == entry[0] and \
            node.ins_order == entry[1]

    def _evict_one(self, protected: set):
        """Evict the LRU unprotected leaf; returns (digest, node) or None."""
        held = []
        victim = None
        heap = self._leaf_heap
        while heap:
            entry = heapq.heappop(heap)
            if not self._valid_leaf(entry):
                continue
            if entry[2] in protected:
                held.append(entry)
                continue
            victim = entry[2]
            break
        for e in held:
            heapq.heappush(heap, e)
        if victim is None:
            return None
        node = self._remove(victim)
        return victim, node

    def _remove(self, d: bytes) -> _Node:
        node = self._blocks.pop(d)
        heapq.heappush(self._free_slots, node.slot)
        if node.parent is not None:
            p = self._blocks[node.parent]
            p.children -= 1
            if node.last_use > p.last_use:  # lazy path stamps (begin_insert)
                p.last_use = node.last_use
            if p.children == 0:
                heapq.heappush(self._leaf_heap, (p.last_use, p.ins_order, node.parent))
        return node

    def check_invariants(self):
        assert self.used_tokens <= self.config.capacity_tokens
        counts: dict = {}
        for d, node in self._blocks.items():
            if node.parent is not None:
                assert node.parent in self._blocks, "prefix closure violated"
                assert self._blocks[node.parent].depth == node.depth - 1
                counts[node.parent] = counts.get(node.parent, 0) + 1
            else:
                assert node.depth == 1
        for d, node in self._blocks.items():
            assert node.children == counts.get(d, 0)
        slots = [n.slot for n in self._blocks.values()]
        assert len(set(slots)) == len(slots), "two blocks share a pool slot"
        assert len(slots) + len(self._free_slots) == self.config.capacity_blocks
        assert not (set(slots) & set(self._free_slots))
        leaves = {d for d, n in self._blocks.items() if n.children == 0}
        live = {e[2] for e in self._leaf_heap if self._valid_leaf(e)}
        assert leaves == live, "leaf heap out of sync"

"""CPU restatement of the reference serving policy — TEST INFRASTRUCTURE ONLY.

Plain-Python restatement (no optimisation) of:
  block_chain            ps/cache.py:39-62      chained blake2b-128 over uint32-LE 16-token blocks
  PrefixCache            ps/cache.py:92-211     binary-search match, suffix-discard insert, O(leaves) LRU scan
  schedule_next / score  ps/scheduling.py:78-136
  Router                 ps/sim.py:52-66
  run (event loop)       ps/sim.py:162-287      with a pluggable service-time function
  p99_nearest_rank       ps/sim.py:146-151
Pinned against fixtures generated from the reference itself (tests/golden/make_golden.py); the product
modules (paper_2505_07203_b200/{cache,scheduling,serving}.py) are checked against this restatement.
"""

from __future__ import annotations

import heapq
import math
from hashlib import blake2b

import numpy as np


def block_chain(tokens, bt: int, base=()) -> list:
    arr = np.ascontiguousarray(tokens, dtype=np.uint32)  # ps/cache.py:51
    chain = list(base)
    prev = chain[-1] if chain else b""
    for i in range(len(chain), len(arr) // bt):  # ps/cache.py:57-61
        prev = blake2b(prev + arr[i * bt:(i + 1) * bt].tobytes(), digest_size=16).digest()
        chain.append(prev)
    return chain


class Block:
    def __init__(self, parent, depth, now, order):
        self.parent, self.depth, self.children, self.last_use, self.ins_order = parent, depth, 0, now, order


class PrefixCache:
    """ps/cache.py:92-211, statement for statement."""

    def __init__(self, capacity_tokens: int, bt: int = 16):
        self.capacity_tokens, self.bt = capacity_tokens, bt
        self.capacity_blocks = capacity_tokens // bt
        self.blocks: dict = {}
        self.leaves: dict = {}
        self.counter = 0

    @property
    def used_tokens(self):
        return len(self.blocks) * self.bt

    def match_chain(self, chain) -> int:  # ps/cache.py:119-130
        if not chain or chain[0] not in self.blocks:
            return 0
        lo, hi = 1, len(chain)
        while lo < hi:
            mid = (lo + hi + 1) // 2
            if chain[mid - 1] in self.blocks:
                lo = mid
            else:
                hi = mid - 1
        return lo * self.bt

    def insert_chain(self, chain, now) -> int:  # ps/cache.py:143-159
        path = set(chain)
        stored = 0
        for i, d in enumerate(chain):
            node = self.blocks.get(d)
            if node is not None:
                node.last_use = now
                stored = i + 1
                continue
            if len(self.blocks) >= self.capacity_blocks and not self.evict_one(path):
                break
            parent = chain[i - 1] if i > 0 else None
            self.counter += 1
            self.blocks[d] = Block(parent, 1 if parent is None else self.blocks[parent].depth + 1, now, self.counter)
            self.leaves[d] = None
            if parent is not None:
                self.blocks[parent].children += 1
                self.leaves.pop(parent, None)
            stored = i + 1
        return stored * self.bt

    def evict_one(self, protected) -> bool:  # ps/cache.py:191-211
        victim, key = None, None
        for d in self.leaves:
            if d in protected:
                continue
            k = (self.blocks[d].last_use, self.blocks[d].ins_order)
            if key is None or k < key:
                victim, key = d, k
        if victim is None:
            return False
        node = self.blocks.pop(victim)
        del self.leaves[victim]
        if node.parent is not None:
            p = self.blocks[node.parent]
            p.children -= 1
            if p.children == 0:
                self.leaves[node.parent] = None
        return True

    def evict_to(self, needed_tokens, protect=()) -> int:  # ps/cache.py:161-173
        if needed_tokens > self.capacity_tokens:
            raise ValueError("cannot free more than the cache capacity")
        protected, freed = set(protect), 0
        while self.capacity_tokens - self.used_tokens < needed_tokens:
            if not self.evict_one(protected):
                raise ValueError("eviction shortfall")
            freed += self.bt
        return freed


def estimate(n_input, n_cached, scoring="proxy", profile=None) -> float:  # ps/scheduling.py:78-86
    if scoring == "proxy":
        return float(n_input - n_cached)
    est = profile[0] * n_input + profile[1] * n_cached + profile[2]  # ps/jct.py:71-76
    return max(0.0, est)


def schedule_next(queue, cache, policy: str, now: float, lam: float = 0.5, scoring="proxy", profile=None):
    """queue entries: dicts with id, n_input, arrival, frozen_jct, chain (ps/scheduling.py:111-136)."""
    if policy == "fifo":
        return min(queue, key=lambda w: (w["arrival"], w["id"]))
    if policy == "srjf":
        return min(queue, key=lambda w: (w["frozen_jct"], w["arrival"], w["id"]))
    return min(queue, key=lambda w: (estimate(w["n_input"], cache.match_chain(w["chain"]), scoring, profile)
                                     - lam * (now - w["arrival"]), w["arrival"], w["id"]))


def p99_nearest_rank(lat) -> float:
    if not lat:
        return 0.0
    s = sorted(lat)
    return s[max(0, math.ceil(0.99 * len(s)) - 1)]


def run(requests, num_instances, policy, capacity_tokens, service_fn, bt=16, lam=0.5, scoring="proxy",
        profile=None):
    """ps/sim.py:162-287 with service_fn(n_input, n_cached) -> seconds. requests: dicts id, user_id, arrival,
    n_input, chain. Returns records as (id, instance, start, completion, n_cached) sorted by completion order."""
    caches = [PrefixCache(capacity_tokens, bt) for _ in range(num_instances)]
    queues = [[] for _ in range(num_instances)]
    busy = [False] * num_instances
    assign, rr = {}, 0
    events, seq = [], 0
    for r in requests:
        heapq.heappush(events, (r["arrival"], 2, seq, r))
        seq += 1
    records = []

    def start_next(i, now):
        nonlocal seq
        w = schedule_next(queues[i], caches[i], policy, now, lam, scoring, profile)
        queues[i].remove(w)
        nc = caches[i].match_chain(w["chain"])
        svc = service_fn(w["n_input"], nc)
        busy[i] = True
        heapq.heappush(events, (now + svc, 1, seq, i))
        seq += 1
        heapq.heappush(events, (now + svc, 0, seq, (i, w, nc, now)))
        seq += 1

    while events:
        now, kind, _, p = heapq.heappop(events)
        if kind == 2:
            i = assign.get(p["user_id"])
            if i is None:
                i = assign[p["user_id"]] = rr % num_instances
                rr += 1
            w = dict(p, arrival=now)
            if policy == "srjf":
                w["frozen_jct"] = estimate(p["n_input"], caches[i].match_chain(p["chain"]), scoring, profile)
            queues[i].append(w)
            if not busy[i]:
                start_next(i, now)
        elif kind == 1:
            busy[p] = False
            if queues[p]:
                start_next(p, now)
        else:
            i, w, nc, started = p
            caches[i].insert_chain(w["chain"], now)
            records.append((w["id"], i, started, now, nc))
    return records

"""Synthetic prefill-only workloads and Poisson arrivals (inputs to the serving benchmarks).

Token streams, per-user lengths and arrival shuffles come from counter-seeded numpy generators keyed
exactly like the reference (ps/workload.py:20-26,113-115), so a (generator, seed) pair yields the same
trace here as there; tests/test_workload_parity.py pins that against golden fixtures. The shape knobs
default to the reference constants (ps/workload.py:27-37) and can be overridden for the BASELINE configs
(e.g. 20k-token post-recommendation prompts, 10k-60k credit documents).
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace
from pathlib import Path
from typing import Sequence

import numpy as np

from .cache import block_chain

# SeedSequence entropy selectors: (trace_seed, stream, index)
STREAM_PROFILE, STREAM_SUFFIX, STREAM_POSTREC_LENGTHS, STREAM_CREDIT_LENGTHS, STREAM_ARRIVALS = range(5)


class WorkloadError(ValueError):
    """Invalid generator parameters or trace file."""


def token_stream(key: Sequence[int], n: int) -> np.ndarray:
    """n uint32 token ids from the generator keyed by `key`."""
    return np.random.default_rng(list(key)).integers(0, 2 ** 32, size=n, dtype=np.uint32)


@dataclass(frozen=True)
class Request:
    """One prefill-only job: a per-user profile prefix plus a request-specific suffix."""

    id: int
    user_id: int
    arrival: float
    profile_len: int
    total_len: int
    seed: int

    @property
    def n_input(self) -> int:
        return self.total_len

    @property
    def profile_tokens(self) -> np.ndarray:
        return token_stream((self.seed, STREAM_PROFILE, self.user_id), self.profile_len)

    @property
    def suffix_tokens(self) -> np.ndarray:
        n = self.total_len - self.profile_len
        if n <= 0:
            return np.empty(0, dtype=np.uint32)
        s = token_stream((self.seed, STREAM_SUFFIX, self.id), n)
        s[0] = np.uint32(self.id)  # siblings diverge right after the shared profile
        return s

    @property
    def tokens(self) -> np.ndarray:
        return np.concatenate([self.profile_tokens, self.suffix_tokens])

    def digest_chain(self, block_tokens: int, memo: dict | None = None) -> list[bytes]:
        """Block digest chain; the profile part is hashed once per (seed, user, length) when memoised."""
        if memo is None or self.profile_len < block_tokens:
            return block_chain(self.tokens, block_tokens)
        key = (self.seed, self.user_id, self.profile_len, block_tokens)
        base = memo.get(key)
        if base is None:
            base = memo[key] = block_chain(self.profile_tokens, block_tokens)
        return block_chain(self.tokens, block_tokens, base=base)


@dataclass(frozen=True, eq=False)
class FixedRequest(Request):
    """A request carrying explicit tokens (worked example, tests)."""

    fixed_tokens: np.ndarray = field(default=None, repr=False)

    @property
    def tokens(self) -> np.ndarray:
        return self.fixed_tokens

    @property
    def profile_tokens(self) -> np.ndarray:
        return self.fixed_tokens

    @property
    def suffix_tokens(self) -> np.ndarray:
        return np.empty(0, dtype=np.uint32)


@dataclass(frozen=True)
class Trace:
    name: str
    seed: int
    requests: tuple

    def __post_init__(self):
        arr = [r.arrival for r in self.requests]
        if any(b < a for a, b in zip(arr, arr[1:])):
            raise WorkloadError("trace arrivals must be nondecreasing")

    @property
    def total_tokens(self) -> int:
        return sum(r.total_len for r in self.requests)

    @property
    def max_request_len(self) -> int:
        return max((r.total_len for r in self.requests), default=0)

    def __len__(self):
        return len(self.requests)


@dataclass(frozen=True)
class PostRecSpec:
    """Post recommendation (ps/workload.py:27-33): users x requests, shared profile + fixed suffix."""

    users: int = 20
    requests_per_user: int = 50
    profile_mean: float = 14_000
    profile_std: float = 3_000
    profile_min: int = 11_000
    profile_max: int = 17_000
    suffix_tokens: int = 150


@dataclass(frozen=True)
class CreditSpec:
    """Credit verification (ps/workload.py:35-37): one long document per user, no sharing."""

    users: int = 60
    min_tokens: int = 40_000
    max_tokens: int = 60_000


# BASELINE.json configs: 20k-token recommendation prompts (19,850 +- 3,000 profile + 150 suffix), U = 40 users
# so 8 GPUs balance under sticky routing; credit documents of 10k-60k tokens.
POSTREC_20K = PostRecSpec(users=40, profile_mean=19_850, profile_min=16_850, profile_max=22_850)
CREDIT_10K_60K = CreditSpec(min_tokens=10_000)


def post_rec_profile_lengths(seed: int, spec: PostRecSpec = PostRecSpec()) -> list[int]:
    rng = np.random.default_rng([seed, STREAM_POSTREC_LENGTHS])
    draws = rng.normal(spec.profile_mean, spec.profile_std, size=spec.users)
    return [int(x) for x in np.clip(np.rint(draws), spec.profile_min, spec.profile_max)]


def credit_lengths(seed: int, spec: CreditSpec = CreditSpec()) -> list[int]:
    rng = np.random.default_rng([seed, STREAM_CREDIT_LENGTHS])
    return [int(x) for x in rng.integers(spec.min_tokens, spec.max_tokens + 1, size=spec.users)]


def gen_post_recommendation(seed: int, spec: PostRecSpec = PostRecSpec()) -> Trace:
    reqs = []
    for user, plen in enumerate(post_rec_profile_lengths(seed, spec)):
        for _ in range(spec.requests_per_user):
            reqs.append(Request(len(reqs), user, 0.0, plen, plen + spec.suffix_tokens, seed))
    return Trace("post-rec", seed, tuple(reqs))


def gen_credit_verification(seed: int, spec: CreditSpec = CreditSpec()) -> Trace:
    reqs = tuple(Request(u, u, 0.0, n, n, seed) for u, n in enumerate(credit_lengths(seed, spec)))
    return Trace("credit", seed, reqs)


def poisson_arrivals(trace: Trace, rate: float, seed: int, keep_sessions: bool = True) -> Trace:
    """Assign Poisson arrivals at `rate` req/s after a seeded shuffle (ps/workload.py:180-207).

    keep_sessions: users arrive as contiguous bursts in a shuffled user order; otherwise requests interleave.
    """
    if rate <= 0:
        raise WorkloadError("rate must be positive")
    rng = np.random.default_rng([seed, STREAM_ARRIVALS])
    reqs = trace.requests
    if keep_sessions:
        users = list(dict.fromkeys(r.user_id for r in reqs))
        perm = rng.permutation(len(users))
        groups: dict = {u: [] for u in users}
        for r in reqs:
            groups[r.user_id].append(r)
        order = [r for k in perm for r in groups[users[k]]]
    else:
        order = [reqs[k] for k in rng.permutation(len(reqs))]
    t = np.cumsum(rng.exponential(1.0 / rate, size=len(reqs)))
    return Trace(trace.name, trace.seed, tuple(replace(r, arrival=float(a)) for r, a in zip(order, t)))


def zero_arrivals(trace: Trace) -> Trace:
    return Trace(trace.name, trace.seed, tuple(replace(r, arrival=0.0) for r in trace.requests))


TRACE_HEADER = "id,user_id,arrival_seconds,profile_len,total_len,seed"


def save_trace(trace: Trace, path):
    rows = [TRACE_HEADER] + [f"{r.id},{r.user_id},{r.arrival!r},{r.profile_len},{r.total_len},{r.seed}"
                             for r in trace.requests]
    Path(path).write_text("\n".join(rows) + "\n", encoding="utf-8")


def load_trace(path, name: str | None = None) -> Trace:
    """Read the reference's line-delimited trace format (ps/workload.py:210-249)."""
    path = Path(path)
    lines = path.read_text(encoding="utf-8").splitlines()
    if not lines or lines[0] != TRACE_HEADER:
        raise WorkloadError(f"{path}: missing trace header")
    reqs, seeds = [], set()
    for no, line in enumerate(lines[1:], start=2):
        if not line.strip():
            continue
        f = line.split(",")
        if len(f) != 6:
            raise WorkloadError(f"{path}:{no}: expected 6 fields")
        reqs.append(Request(int(f[0]), int(f[1]), float(f[2]), int(f[3]), int(f[4]), int(f[5])))
        seeds.add(int(f[5]))
    return Trace(name or path.stem, seeds.pop() if len(seeds) == 1 else 0, tuple(reqs))


def worked_example() -> tuple[Trace, int]:
    """Four simultaneous requests A<C<B<D (A prefix of D, C prefix of B) and a 2048-token cache.

    The paper's scheduling example (ps/workload.py:252-283): cache hits fifo=1,
    srjf=1, srjf-calibrated=2 with calibrated order A, D, C, B.
    """
    la, lc, lb, ld = 1024, 2048, 2560, 2944
    seed = 7
    ad = token_stream((seed, 10, 0), ld)
    cb = token_stream((seed, 10, 1), lb)
    toks = {0: ad[:la], 1: cb[:lb], 2: cb[:lc], 3: ad[:ld]}
    reqs = tuple(FixedRequest(rid, 0 if rid in (0, 3) else 1, 0.0, len(t), len(t), seed, fixed_tokens=t)
                 for rid, t in toks.items())
    return Trace("worked-example", seed, reqs), 2048

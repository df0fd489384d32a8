"""Engine: the reference-facing request API over the C-ABI (one engine per GPU).

The reference has no request API; the paper describes it (submit a prompt plus an allowed-token list,
get the constrained next-token choice and its probabilities). The engine slot it
fills is `execute_time(variant, geom, gpu, params, n_input, n_cached)` (ps/costs.py:259-280), called
from sim.run.start_next (ps/sim.py:217-220): `Engine.prefill` runs the real forward and reports the
measured device seconds in place of the modelled service time.

Error mapping mirrors the reference taxonomy: PO_ERR_CAPACITY -> CapacityError (ps/costs.py:40-45),
PO_ERR_CONFIG -> ConfigError (GeometryError / NumericsError analogue).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib
from .config import BLOCK_TOKENS, DEFAULT_CHUNK, ModelConfig, get_preset, to_c_cfg


class CapacityError(ValueError):
    """Request longer than the engine's maximum input length (ps/costs.py:40-45)."""


class ConfigError(ValueError):
    """Invalid model/engine configuration (ps/geometry.py:18-23 analogue)."""


@dataclass(frozen=True)
class PrefillResult:
    """Outcome of one prefill-only request."""

    token: int  # the chosen allowed token id
    index: int  # its position in the allowed list
    probs: np.ndarray  # softmax restricted to the allowed ids
    logits: np.ndarray  # raw logits of the allowed ids
    n_cached: int  # prefix tokens served from the pool (reference accounting)
    service_s: float  # device seconds of the forward (replaces execute_time)


def _raise(err: _lib.PrefillOnlyError):
    if err.code == _lib.PO_ERR_CAPACITY:
        raise CapacityError(str(err)) from None
    if err.code == _lib.PO_ERR_CONFIG:
        raise ConfigError(str(err)) from None
    raise err


@dataclass(frozen=True)
class Ticket:
    """An enqueued request (Engine.prefill_submit)."""

    id: int
    allowed: np.ndarray
    n_cached: int


class Engine:
    """One GPU's PrefillOnly engine: weights, arena, one-layer KV buffer and the prefix-KV pool."""

    def __init__(self, model: ModelConfig | str = "llama-3.1-8b", device: int = 0, seed: int = 0,
                 max_tokens: int = 32_768, chunk: int = DEFAULT_CHUNK, block_tokens: int = BLOCK_TOKENS,
                 pool_blocks: int = -1, pool_mem_fraction: float = 0.9, last_row_only: bool = True):
        self.model = get_preset(model) if isinstance(model, str) else model
        self.device = device
        self.seed = seed
        self.max_tokens = max_tokens
        self.chunk = chunk
        self.block_tokens = block_tokens
        lib = _lib.load()
        self.last_row_only = last_row_only
        cfg = to_c_cfg(self.model, max_tokens, chunk, block_tokens, pool_blocks, pool_mem_fraction, last_row_only)
        handle = ctypes.c_void_p()
        try:
            _lib.check(lib.po_init(device, ctypes.addressof(cfg), seed, ctypes.addressof(handle)))
        except _lib.PrefillOnlyError as err:
            _raise(err)
        self._h = handle
        info = (ctypes.c_int64 * 8)()
        _lib.check(lib.po_engine_info(self._h, ctypes.addressof(info), 8))
        self.pool_blocks = int(info[0])
        self.weight_bytes = int(info[1])
        self.arena_bytes = int(info[2])
        self.pool_bytes = int(info[3])
        self.block_bytes = int(info[4])
        self.free_bytes_after_init = int(info[6])
        self.workspace_bytes = int(info[7])

    # ------------------------------------------------------------------ lifecycle
    def close(self):
        if getattr(self, "_h", None):
            _lib.load().po_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def capacity_tokens(self) -> int:
        """Prefix-pool capacity in tokens (CacheConfig.capacity_tokens, ps/cache.py:65-80)."""
        return self.pool_blocks * self.block_tokens

    # ------------------------------------------------------------------ requests
    def prefill(self, tokens, allowed: Sequence[int], n_cached: int = 0,
                pool_block_ids: Sequence[int] | None = None, stream: int | None = None) -> PrefillResult:
        """Run one prefill-only request; returns the allowed-token choice and its probabilities.

        tokens: uint32 ids (embedded as id % vocab). n_cached: block-aligned prefix already in the pool,
        with pool_block_ids[b] its slots; later entries of pool_block_ids are admission slots (-1 = discard).
        """
        return self.prefill_wait(self.prefill_submit(tokens, allowed, n_cached, pool_block_ids, stream))

    def prefill_submit(self, tokens, allowed: Sequence[int], n_cached: int = 0,
                       pool_block_ids: Sequence[int] | None = None, stream: int | None = None) -> "Ticket":
        """Stage and enqueue one request (po_prefill_submit); returns at once with a ticket for prefill_wait.
        At most three tickets may be outstanding per engine (the staging ring has four entries)."""
        toks = np.ascontiguousarray(tokens, dtype=np.uint32)
        alw = np.ascontiguousarray(allowed, dtype=np.int32)
        n = int(toks.shape[0])
        ids = np.ascontiguousarray(pool_block_ids if pool_block_ids is not None else [], dtype=np.int32)
        t = ctypes.c_int64(0)
        rc = _lib.load().po_prefill_submit(self._h, toks.ctypes.data, n, int(n_cached), alw.ctypes.data, len(alw),
                                           ids.ctypes.data if len(ids) else None, len(ids), ctypes.addressof(t),
                                           stream)
        try:
            _lib.check(rc)
        except _lib.PrefillOnlyError as err:
            _raise(err)
        return Ticket(int(t.value), alw, int(n_cached))

    def prefill_done(self, ticket: "Ticket") -> bool:
        """Non-blocking: has the ticket's forward completed (po_prefill_query)?"""
        done = ctypes.c_int32(0)
        _lib.call("po_prefill_query", self._h, ticket.id, ctypes.addressof(done))
        return bool(done.value)

    def prefill_wait(self, ticket: "Ticket") -> PrefillResult:
        """Block until the ticket's forward completed and return its result (po_prefill_wait)."""
        alw = ticket.allowed
        logits = np.empty(len(alw), dtype=np.float32)
        probs = np.empty(len(alw), dtype=np.float32)
        argmax = ctypes.c_int32(-1)
        ms = ctypes.c_float()
        rc = _lib.load().po_prefill_wait(self._h, ticket.id, logits.ctypes.data, probs.ctypes.data,
                                         ctypes.addressof(argmax), ctypes.addressof(ms))
        try:
            _lib.check(rc)
        except _lib.PrefillOnlyError as err:
            _raise(err)
        idx = int(argmax.value)
        return PrefillResult(token=int(alw[idx]), index=idx, probs=probs, logits=logits, n_cached=ticket.n_cached,
                             service_s=float(ms.value) * 1e-3)

    def prefill_device(self, d_tokens: int, n: int, d_allowed: int, n_allowed: int, d_logits: int, d_probs: int,
                       d_argmax: int, n_cached: int = 0, pool_block_ids: Sequence[int] | None = None,
                       stream: int | None = None):
        """Asynchronous forward on device-resident inputs/outputs (raw device pointers)."""
        ids = np.ascontiguousarray(pool_block_ids if pool_block_ids is not None else [], dtype=np.int32)
        rc = _lib.load().po_prefill_device(self._h, d_tokens, n, int(n_cached), d_allowed, n_allowed,
                                           ids.ctypes.data if len(ids) else None, len(ids), d_logits, d_probs,
                                           d_argmax, stream)
        try:
            _lib.check(rc)
        except _lib.PrefillOnlyError as err:
            _raise(err)

    @property
    def stream(self) -> int:
        """The engine's CUDA stream handle (cudaStream_t as int)."""
        out = ctypes.c_void_p()
        _lib.call("po_engine_stream", self._h, ctypes.addressof(out))
        return int(out.value or 0)

    @property
    def last_launches(self) -> int:
        out = ctypes.c_int32()
        _lib.call("po_last_launches", self._h, ctypes.addressof(out))
        return int(out.value)

    KERNEL_CLASSES = ("embed", "rmsnorm", "kv_gather", "gemm_qkv_rope", "kv_scatter", "attention",
                      "gemm_o_resid", "gemm_gate_up_silu", "gemm_down_resid", "lm_head", "stream_layer", "mlp_fused")

    def profile_begin(self):
        _lib.call("po_profile_begin", self._h)

    def profile_end(self) -> dict:
        """{class: (milliseconds, launches)} accumulated since profile_begin (CUDA events, engine stream)."""
        k = len(self.KERNEL_CLASSES)
        ms = (ctypes.c_float * k)()
        cnt = (ctypes.c_int32 * k)()
        _lib.call("po_profile_end", self._h, ctypes.addressof(ms), ctypes.addressof(cnt), k)
        return {name: (float(ms[i]), int(cnt[i])) for i, name in enumerate(self.KERNEL_CLASSES)}

    def load_weight(self, kind: int, layer: int, array: np.ndarray):
        """Overwrite one weight tensor (logical layout; see po_load_weight)."""
        arr = np.ascontiguousarray(array)
        _lib.call("po_load_weight", self._h, kind, layer, arr.ctypes.data, arr.size)

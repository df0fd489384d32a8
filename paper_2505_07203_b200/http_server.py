"""HTTP front end for prefill-only requests (the paper's OpenAI-style entry point,
PAPER.md:403-409). The reference has no server; this is a thin FastAPI layer over serving.Server.submit.

  POST /v1/prefill   {"user_id": 7, "tokens": [...]  or  "prompt": "...", "allowed": [9642, 2822]}
               ->    {"token": 9642, "index": 0, "probs": [...], "logits": [...], "n_cached": 19840,
                      "latency_s": 0.013, "service_s": 0.012}
  GET  /v1/stats     served requests, mean / p99 latency, prefix-hit counts (RequestRecord fields)

OpenAI-compatible surface (the paper's vLLM-based front end speaks the OpenAI API; prefill-only means exactly one
generated token, chosen among the allowed ids):
  POST /v1/completions  {"model": "...", "prompt": "..." | [ids], "max_tokens": 1,
                         "allowed_token_ids": [9642, 2822]  (vLLM's SamplingParams name)
                         or "logit_bias": {"9642": 100, "2822": 100}  (the OpenAI way: ids with a bias >= 100
                         are the allowed set), "logprobs": k, "user": "..."}
                     -> {"object": "text_completion", "choices": [{"text", "token_ids", "logprobs", "finish_reason"}],
                         "usage": {"prompt_tokens", "completion_tokens": 1, "prompt_tokens_details": {"cached_tokens"}}}
  GET  /v1/models

Text prompts go through `--tokenizer PATH` (a local Hugging Face tokenizer directory, e.g. the model's own) when
given; none ship offline, so by default "prompt" text is encoded as its UTF-8 bytes (token id = byte), which is
enough for prefix sharing to behave like real prompts; pass "tokens" for real tokenizer ids.

  python -m paper_2505_07203_b200.http_server --gpus 1 --model llama-3.1-8b --port 8000
"""

from __future__ import annotations

import argparse
import itertools
import threading
import time

import numpy as np


class _HttpRequest:
    """Request duck type for the scheduler: .id, .user_id, .n_input, .tokens (pkg/tests/test_scheduler.py:15-20)."""

    __slots__ = ("id", "user_id", "tokens", "n_input")

    def __init__(self, rid: int, user_id: int, tokens: np.ndarray):
        self.id = rid
        self.user_id = user_id
        self.tokens = tokens
        self.n_input = int(tokens.shape[0])


try:  # pydantic / fastapi are optional at import time (the engine does not need them)
    from pydantic import BaseModel

    class PrefillBody(BaseModel):
        user_id: int = 0
        tokens: list[int] | None = None
        prompt: str | None = None
        allowed: list[int]
    class CompletionBody(BaseModel):
        model: str | None = None
        prompt: str | list[int]
        max_tokens: int = 1
        allowed_token_ids: list[int] | None = None
        logit_bias: dict[str, float] | None = None
        logprobs: int | None = None
        user: str | int | None = None
except ImportError:  # pragma: no cover
    PrefillBody = None
    CompletionBody = None


class ByteTokenizer:
    """Offline stand-in: a prompt's UTF-8 bytes are its token ids; byte ids decode as their byte, others as <id>."""

    def encode(self, text: str) -> list:
        return list(text.encode("utf-8"))

    def decode_one(self, tid: int) -> str:
        return bytes([tid]).decode("latin-1") if 0 <= tid < 256 else f"<{tid}>"


class HfTokenizer:
    """A Hugging Face tokenizer loaded from local files (tokenizer.json / tokenizer.model directory, e.g. the
    model's own): `--tokenizer PATH`. No special tokens are added, so a prompt's ids are exactly its text."""

    def __init__(self, path: str):
        from transformers import AutoTokenizer

        self.tok = AutoTokenizer.from_pretrained(path, local_files_only=True)

    def encode(self, text: str) -> list:
        return list(self.tok.encode(text, add_special_tokens=False))

    def decode_one(self, tid: int) -> str:
        return self.tok.decode([tid])


_TOKENIZER = ByteTokenizer()


def _token_text(tid: int) -> str:
    return _TOKENIZER.decode_one(tid)


def create_app(server, tokenizer=None):
    global _TOKENIZER
    if tokenizer is not None:
        _TOKENIZER = tokenizer
    from fastapi import FastAPI, HTTPException

    from . import _lib
    from ._lib import PrefillOnlyError

    app = FastAPI(title="prefillonly-b200")
    ids = itertools.count()
    lock = threading.Lock()

    @app.post("/v1/prefill")
    def prefill(body: PrefillBody):
        if body.tokens is None and body.prompt is None:
            raise HTTPException(400, "need tokens or prompt")
        if not body.allowed:
            raise HTTPException(400, "allowed must be non-empty")
        raw = body.tokens if body.tokens is not None else _TOKENIZER.encode(body.prompt)
        if not raw:
            raise HTTPException(400, "empty prompt")
        if min(raw) < 0 or max(raw) >= 2 ** 32:
            raise HTTPException(400, "token ids must be in [0, 2^32)")
        vocab = server.workers[0].engine.model.vocab if hasattr(server.workers[0].engine, "model") else None
        if min(body.allowed) < 0 or (vocab is not None and max(body.allowed) >= vocab):
            raise HTTPException(400, f"allowed ids must be in [0, {vocab})")
        toks = np.asarray(raw, dtype=np.uint32)
        with lock:
            rid = next(ids)
        t0 = time.perf_counter()
        try:
            res = server.submit(_HttpRequest(rid, body.user_id, toks), body.allowed).result()
        except ValueError as err:  # CapacityError / ConfigError
            raise HTTPException(413 if "exceeds" in str(err) else 400, str(err)) from None
        except PrefillOnlyError as err:  # C-ABI status: request errors are the client's, the rest the server's
            client = err.code in (_lib.PO_ERR_ARG, _lib.PO_ERR_POOL)
            raise HTTPException(400 if client else 500, str(err)) from None
        return {"id": rid, "token": res.token, "index": res.index, "probs": res.probs.tolist(),
                "logits": res.logits.tolist(), "n_cached": res.n_cached,
                "latency_s": time.perf_counter() - t0, "service_s": res.service_s}

    model_name = getattr(getattr(server.workers[0].engine, "model", None), "name", "prefillonly")
    users: dict = {}

    @app.get("/v1/models")
    def models():
        return {"object": "list", "data": [{"id": model_name, "object": "model", "owned_by": "prefillonly-b200"}]}

    @app.post("/v1/completions")
    def completions(body: CompletionBody):
        if body.max_tokens != 1:
            raise HTTPException(400, "prefill-only serving produces exactly one token: max_tokens must be 1")
        allowed = body.allowed_token_ids
        if allowed is None and body.logit_bias:
            allowed = [int(k) for k, v in body.logit_bias.items() if v >= 100]
        if not allowed:
            raise HTTPException(400, "give allowed_token_ids, or logit_bias with +100 on the allowed ids")
        raw = body.prompt if isinstance(body.prompt, list) else _TOKENIZER.encode(body.prompt)
        if not raw:
            raise HTTPException(400, "empty prompt")
        if min(raw) < 0 or max(raw) >= 2 ** 32:
            raise HTTPException(400, "token ids must be in [0, 2^32)")
        vocab = getattr(getattr(server.workers[0].engine, "model", None), "vocab", None)
        if min(allowed) < 0 or (vocab is not None and max(allowed) >= vocab):
            raise HTTPException(400, f"allowed ids must be in [0, {vocab})")
        with lock:
            rid = next(ids)
            uid = users.setdefault(body.user, len(users)) if body.user is not None else rid
        try:
            res = server.submit(_HttpRequest(rid, uid, np.asarray(raw, dtype=np.uint32)), allowed).result()
        except ValueError as err:
            raise HTTPException(413 if "exceeds" in str(err) else 400, str(err)) from None
        except PrefillOnlyError as err:
            raise HTTPException(400 if err.code in (_lib.PO_ERR_ARG, _lib.PO_ERR_POOL) else 500, str(err)) from None
        logp = np.log(np.maximum(res.probs.astype(np.float64), 1e-45))
        choice = {"index": 0, "text": _token_text(res.token), "token_ids": [res.token], "finish_reason": "length"}
        if body.logprobs:
            order = np.argsort(-logp, kind="stable")[: body.logprobs]
            choice["logprobs"] = {"tokens": [_token_text(res.token)], "token_logprobs": [float(logp[res.index])],
                                  "top_logprobs": [{_token_text(allowed[i]): float(logp[i]) for i in order}],
                                  "allowed_token_ids": list(allowed), "allowed_probs": res.probs.tolist()}
        n = len(raw)
        return {"id": f"cmpl-{rid}", "object": "text_completion", "created": int(time.time()), "model": model_name,
                "choices": [choice],
                "usage": {"prompt_tokens": n, "completion_tokens": 1, "total_tokens": n + 1,
                          "prompt_tokens_details": {"cached_tokens": res.n_cached}}}

    @app.get("/v1/stats")
    def stats():
        rep = server.report()
        return {"served": rep.served, "mean_latency_s": rep.mean_latency, "p99_latency_s": rep.p99_latency,
                "cache_hit_requests": rep.cache_hit_requests, "cache_hit_tokens": rep.cache_hit_tokens}

    return app


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--model", default="llama-3.1-8b")
    ap.add_argument("--max-tokens", type=int, default=32768)
    ap.add_argument("--host", default="127.0.0.1")
    ap.add_argument("--port", type=int, default=8000)
    ap.add_argument("--tokenizer", default=None,
                    help="local Hugging Face tokenizer directory for text prompts (default: UTF-8 bytes as ids)")
    ap.add_argument("--routing", default="round_robin", choices=["round_robin", "least_work"],
                    help="first-seen user placement across GPUs: the reference's round robin, or least outstanding "
                         "cache-miss work (SURVEY H9)")
    args = ap.parse_args()
    import uvicorn

    from .engine import Engine
    from .scheduling import Policy
    from .serving import Server

    engines = [Engine(args.model, device=d, max_tokens=args.max_tokens) for d in range(args.gpus)]
    srv = Server(engines, Policy.srjf_calibrated(), routing=args.routing)
    tok = HfTokenizer(args.tokenizer) if args.tokenizer else None
    uvicorn.run(create_app(srv, tok), host=args.host, port=args.port)


if __name__ == "__main__":
    main()

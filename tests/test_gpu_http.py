"""The HTTP front end (OpenAI-compatible /v1/completions and /v1/prefill) over a real GPU Engine.

Requests go through FastAPI -> serving.Server -> Engine.prefill (C-ABI, tcgen05 forward); the answers must equal the
CPU oracle's, and a second request of the same user must be served from the prefix pool.
"""

import numpy as np
import pytest

from oracle import llama_ref
from paper_2505_07203_b200.config import TINY
from paper_2505_07203_b200.engine import Engine
from paper_2505_07203_b200.scheduling import Policy
from paper_2505_07203_b200.serving import Server

fastapi = pytest.importorskip("fastapi")
from fastapi.testclient import TestClient  # noqa: E402

from paper_2505_07203_b200.http_server import create_app  # noqa: E402

pytestmark = pytest.mark.gpu
YES_NO = [9642, 2822]


def test_openai_completions_on_gpu_match_oracle():
    cfg = llama_ref.Cfg.from_model(TINY)
    w = llama_ref.make_weights(cfg, 42)
    profile = np.random.default_rng([5, 0, 0]).integers(0, 32000, size=1500).tolist()
    with Engine(TINY, seed=42, max_tokens=4096, chunk=1024, pool_blocks=512) as eng:
        srv = Server([eng], Policy.srjf_calibrated())
        try:
            client = TestClient(create_app(srv))
            for k, suffix in enumerate(([11, 12, 13] * 20, [21, 22] * 40)):
                prompt = profile + suffix
                r = client.post("/v1/completions", json={"prompt": prompt, "max_tokens": 1,
                                                         "allowed_token_ids": YES_NO, "logprobs": 2,
                                                         "user": "u1"})
                assert r.status_code == 200, r.text
                body = r.json()
                logits, probs, am = llama_ref.llama_forward(cfg, w, np.asarray(prompt, dtype=np.uint32), YES_NO)
                assert body["choices"][0]["token_ids"] == [YES_NO[am]]
                got = np.asarray(body["choices"][0]["logprobs"]["allowed_probs"])
                assert np.abs(got - probs).max() < 5e-3
                cached = body["usage"]["prompt_tokens_details"]["cached_tokens"]
                assert cached == (0 if k == 0 else 1488)  # second request: the shared profile blocks (93 x 16)
            r = client.post("/v1/prefill", json={"user_id": 3, "tokens": profile, "allowed": YES_NO})
            assert r.status_code == 200 and r.json()["token"] in YES_NO
        finally:
            srv.close()

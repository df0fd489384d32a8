"""Persistent weight-streaming kernel (csrc/stream.cu, po_op_stream_gemm) against an fp32 torch reference.

The kernel runs the prefix-hit path's layer GEMMs (M <= 256 miss rows): the (weight tile, k-block) space of every phase
is cut into equal ranges over the SM pairs, split tiles are fixed up in-kernel, and a second phase consumes the first
one's output across a grid barrier. Shapes cover a tile cut into more segments than the pair count allows (W < pairs),
the Llama-3.1-8B hit shapes (QKV / O / gate-up / down at M = 160), M = 1 and M = 129 (second CTA of each pair partly
empty), and two-phase chains. Tolerance: bf16 output rounding of an fp32-accumulated product.
"""

import ctypes

import pytest

torch = pytest.importorskip("torch")

from paper_2505_07203_b200 import _lib  # noqa: E402

pytestmark = pytest.mark.gpu


def _p(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def run(A, B1, B2=None):
    M, K = A.shape
    N1 = B1.shape[0]
    out1 = torch.empty(M, N1, dtype=torch.bfloat16, device="cuda")
    out2 = torch.empty(M, B2.shape[0], dtype=torch.bfloat16, device="cuda") if B2 is not None else None
    _lib.call("po_op_stream_gemm", _p(A), A.stride(0), _p(B1), B1.stride(0), _p(out1), out1.stride(0), M, N1, K,
              _p(B2), B2.stride(0) if B2 is not None else 0, _p(out2), out2.stride(0) if B2 is not None else 0,
              B2.shape[0] if B2 is not None else 0, None)
    torch.cuda.synchronize()
    return out1, out2


def close(out, ref):
    err = (out.float() - ref).abs().max().item()
    scale = ref.abs().max().item()
    assert err <= 1e-2 * scale + 1e-3, (err, scale)


@pytest.mark.parametrize("M,N,K", [(1, 256, 256), (100, 512, 256), (129, 1024, 1024), (160, 6144, 4096),
                                   (160, 4096, 4096), (160, 28672, 4096), (160, 4096, 14336), (256, 2048, 512)])
def test_stream_gemm_matches_torch(M, N, K):
    torch.manual_seed(M * 7 + N + K)
    A = (torch.randn(M, K, device="cuda")).to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    out, _ = run(A, B)
    close(out, A.float() @ B.float().T)


@pytest.mark.parametrize("M,N1,K,N2", [(160, 4096, 4096, 4096), (1, 2048, 256, 256), (200, 1024, 1024, 512)])
def test_stream_two_phase_chain(M, N1, K, N2):
    torch.manual_seed(M + N1 + N2)
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B1 = (torch.randn(N1, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    B2 = (torch.randn(N2, N1, device="cuda") / N1 ** 0.5).to(torch.bfloat16)
    o1, o2 = run(A, B1, B2)
    r1 = A.float() @ B1.float().T
    close(o1, r1)
    close(o2, o1.float() @ B2.float().T)


def test_stream_gemm_repeatable():
    """Fixed segment order: the same launch twice gives bit-identical outputs."""
    torch.manual_seed(3)
    A = torch.randn(160, 4096, device="cuda").to(torch.bfloat16)
    B = (torch.randn(4096, 4096, device="cuda") / 64).to(torch.bfloat16)
    a, _ = run(A, B)
    b, _ = run(A, B)
    assert torch.equal(a, b)


def test_engine_with_streaming_kernel_matches_oracle():
    """The engine's opt-in streaming path (PO_STREAM=1: prefix hits' layer GEMMs as phases of stream_kernel) gives the
    oracle's answers, in a fresh process (the switch is read once per process)."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    code = r'''
import numpy as np
from oracle import llama_ref
from paper_2505_07203_b200.config import ModelConfig
from paper_2505_07203_b200.engine import Engine
SMALL = ModelConfig("small", 2, 1024, 8, 2, 128, 2816, 4096)
cfg = llama_ref.Cfg.from_model(SMALL)
w = llama_ref.make_weights(cfg, 7)
toks = np.random.default_rng([70, 0, 0]).integers(0, 2 ** 32, size=1600, dtype=np.uint32)
slots = list(range(100))
with Engine(SMALL, seed=7, max_tokens=2048, chunk=1024, pool_blocks=256) as e:
    e.prefill(toks[:1344], [5, 11, 4095], 0, slots[:84])
    for nc, n in ((1344, 1504), (1344, 1600), (1584, 1600), (0, 200), (0, 1)):
        res = e.prefill(toks[:n], [5, 11, 4095], nc, slots[: n // 16])
        logits, _, am = llama_ref.llama_forward(cfg, w, toks[:n], [5, 11, 4095])
        err = np.abs(res.logits - logits).max()
        assert err <= 1e-2 + 5e-3 * np.abs(logits).max(), (n, nc, err)
        assert res.index == am, (n, nc)
print("ok")
'''
    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, PO_STREAM="1", PYTHONPATH=str(root))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]

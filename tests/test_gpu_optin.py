"""Opt-in kernel paths against the same references as the default path, each in a child process (the switches are
read once per process):
  * PO_SK=1: stream-K short-launch GEMMs (csrc/gemm_sk.cu) - the short-M GEMM tests (fp32 torch reference of each
    epilogue) and the engine tests (CPU oracle: argmax identical, logits within the bf16 tolerance);
  * PO_SK_RED=1: stream-K with split-K-reduce epilogues for the residual / RoPE short launches - the same tests;
  * PO_FUSED_MLP=1: the fused per-layer MLP launch (csrc/mlp.cu) - the engine tests (including the bit-exact chunk
    invariance across 512 / 1024 / 8192-row chunks) and the Llama-3.1-8B-dims oracle fixtures."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _run(args, **switches):
    env = dict(os.environ, **switches)
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", *args], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]


def test_stream_k_short_gemms():
    _run(["tests/test_gpu_gemm.py", "-k", "swap or splitk"], PO_SK="1")
    _run(["tests/test_gpu_gemm.py", "-k", "swap or splitk"], PO_SK="0")


def test_stream_k_engine_against_oracle():
    _run(["tests/test_gpu_engine.py", "tests/test_gpu_parity_fullsize.py"], PO_SK="1")


def test_stream_k_reduce_mode():
    _run(["tests/test_gpu_gemm.py", "-k", "swap or splitk"], PO_SK_RED="1")
    _run(["tests/test_gpu_engine.py", "tests/test_gpu_parity_fullsize.py"], PO_SK_RED="1")


def test_fused_mlp_engine_against_oracle():
    _run(["tests/test_gpu_engine.py", "tests/test_gpu_parity_fullsize.py", "tests/test_gpu_fullsize.py"],
         PO_FUSED_MLP="1")

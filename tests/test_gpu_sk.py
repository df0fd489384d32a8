"""The opt-in stream-K short-launch GEMM (PO_SK=1, csrc/gemm_sk.cu) against the same references as the default path:
the short-M GEMM tests (fp32 torch reference of each epilogue) and the engine tests (CPU oracle: argmax identical,
logits within the bf16 tolerance), run in a child process because the switch is read once per process."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _run(args):
    env = dict(os.environ, PO_SK="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", *args], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]


def test_stream_k_short_gemms():
    _run(["tests/test_gpu_gemm.py", "-k", "swap or splitk"])


def test_stream_k_engine_against_oracle():
    _run(["tests/test_gpu_engine.py", "tests/test_gpu_parity_fullsize.py"])

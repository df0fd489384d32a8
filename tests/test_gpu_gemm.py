"""tcgen05 GEMM parity (po_op_gemm) against an fp32 torch reference of the same op.

The chunked matmuls of block_forward_hybrid (ps/numerics.py:236-239,244-255,259-274) are the
reference stages these epilogues fuse; for a floating-point kernel the task's rule is a plain
fp32 reference of the same op, with the tolerance written here.
"""

import ctypes

import pytest

torch = pytest.importorskip("torch")

from paper_2505_07203_b200 import _lib  # noqa: E402

pytestmark = pytest.mark.gpu

# bf16 output rounding (2^-8 relative) + fp32 accumulation-order noise
TOL_BF16 = 1.5e-2
TOL_F32 = 2e-3


def _p(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-30)).item()


def _gemm(A, B, out=None, resid=None, epi=_lib.EPI_BF16, rope=None, pos_offset=0, rope_cols=0):
    M, K = A.shape
    N = B.shape[0]
    ldo = out.stride(0) if out is not None else 0
    ldr = resid.stride(0) if resid is not None else 0
    _lib.call("po_op_gemm", _p(A), A.stride(0), _p(B), B.stride(0), _p(out), ldo, _p(resid), ldr,
              M, N, K, epi, _p(rope), pos_offset, rope_cols, None)
    torch.cuda.synchronize()


def _rand(*shape, scale=1.0):
    return (torch.randn(*shape, device="cuda") * scale).to(torch.bfloat16)


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (300, 512, 256), (2048, 1024, 4096), (777, 6144, 512),
                                   (4096, 4096, 4096)])
def test_gemm_bf16(M, N, K):
    torch.manual_seed(M + N + K)
    A = _rand(M, K)
    B = _rand(N, K, scale=K ** -0.5)
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    _gemm(A, B, out)
    ref = A.float() @ B.float().T
    assert _rel(out, ref) < TOL_BF16


def test_gemm_f32_exactish():
    torch.manual_seed(1)
    M, N, K = 513, 768, 1024
    A = _rand(M, K)
    B = _rand(N, K, scale=K ** -0.5)
    out = torch.empty(M, N, dtype=torch.float32, device="cuda")
    _gemm(A, B, out, epi=_lib.EPI_F32)
    ref = A.float() @ B.float().T
    assert _rel(out, ref) < TOL_F32


def test_gemm_resid_inplace():
    torch.manual_seed(2)
    M, N, K = 1000, 512, 1024
    A = _rand(M, K)
    B = _rand(N, K, scale=K ** -0.5)
    resid = torch.randn(M, N, device="cuda")
    base = resid.clone()
    _gemm(A, B, resid=resid, epi=_lib.EPI_RESID_F32)
    ref = base + A.float() @ B.float().T
    assert _rel(resid, ref) < TOL_F32


def test_gemm_silu_mul_interleaved():
    torch.manual_seed(3)
    M, I, K = 640, 512, 256
    A = _rand(M, K)
    gate = _rand(I, K, scale=K ** -0.5)
    up = _rand(I, K, scale=K ** -0.5)
    # interleave by 16-row groups: [g0..g15, u0..u15, g16..g31, u16..u31, ...]
    W = torch.stack([gate.view(I // 16, 16, K), up.view(I // 16, 16, K)], dim=1).reshape(2 * I, K).contiguous()
    out = torch.empty(M, I, dtype=torch.bfloat16, device="cuda")
    _gemm(A, W, out, epi=_lib.EPI_SILU_MUL)
    g = A.float() @ gate.float().T
    u = A.float() @ up.float().T
    ref = g / (1 + torch.exp(-g)) * u
    assert _rel(out, ref) < TOL_BF16


def test_gemm_qkv_rope():
    torch.manual_seed(4)
    M, K = 300, 256
    nq, nkv, hd = 2, 1, 128
    N = (nq + 2 * nkv) * hd
    A = _rand(M, K)
    B = _rand(N, K, scale=K ** -0.5)
    pos_offset = 37
    pos = torch.arange(pos_offset + M, dtype=torch.float32)
    inv = 1.0 / (10000.0 ** (torch.arange(0, hd, 2, dtype=torch.float32) / hd))
    ang = pos[:, None] * inv[None, :]
    table = torch.stack([torch.cos(ang), torch.sin(ang)], dim=-1).contiguous().cuda()  # [pos, 64, 2]
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    rope_cols = (nq + nkv) * hd
    _gemm(A, B, out, epi=_lib.EPI_QKV_ROPE, rope=table, pos_offset=pos_offset, rope_cols=rope_cols)
    y = (A.float() @ B.float().T).view(M, -1, hd)
    c = table[pos_offset:pos_offset + M, :, 0][:, None, :]
    s = table[pos_offset:pos_offset + M, :, 1][:, None, :]
    x1, x2 = y[..., :64], y[..., 64:]
    rot = torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)
    heads_rot = rope_cols // hd
    ref = torch.cat([rot[:, :heads_rot], y[:, heads_rot:]], dim=1).reshape(M, N)
    assert _rel(out, ref) < TOL_BF16


def test_gemm_rejects_bad_shape():
    A = _rand(64, 64)
    B = _rand(100, 64)
    out = torch.empty(64, 100, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(_lib.PrefillOnlyError):
        _gemm(A, B, out)


# ---- split-K path (small M, long K: prefix-hit requests); partials summed in a fixed order, then the epilogue
@pytest.mark.parametrize("M,N,K", [(160, 6144, 4096), (1, 4096, 4096), (150, 4096, 14336), (300, 1024, 8192)])
def test_splitk_bf16_and_resid(M, N, K):
    torch.manual_seed(M + K)
    A = _rand(M, K)
    B = _rand(N, K, scale=K ** -0.5)
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    _gemm(A, B, out)
    ref = A.float() @ B.float().T
    assert _rel(out, ref) < TOL_BF16
    resid = torch.randn(M, N, device="cuda")
    base = resid.clone()
    _gemm(A, B, resid=resid, epi=_lib.EPI_RESID_F32)
    assert _rel(resid, base + ref) < TOL_F32


def test_splitk_silu_mul():
    torch.manual_seed(8)
    M, I, K = 150, 2048, 4096
    A = _rand(M, K)
    gate = _rand(I, K, scale=K ** -0.5)
    up = _rand(I, K, scale=K ** -0.5)
    W = torch.stack([gate.view(I // 16, 16, K), up.view(I // 16, 16, K)], dim=1).reshape(2 * I, K).contiguous()
    out = torch.empty(M, I, dtype=torch.bfloat16, device="cuda")
    _gemm(A, W, out, epi=_lib.EPI_SILU_MUL)
    g = A.float() @ gate.float().T
    u = A.float() @ up.float().T
    assert _rel(out, g / (1 + torch.exp(-g)) * u) < TOL_BF16


def test_splitk_qkv_rope():
    torch.manual_seed(9)
    M, K, hd = 150, 4096, 128
    nq, nkv = 8, 2
    N = (nq + 2 * nkv) * hd
    A = _rand(M, K)
    B = _rand(N, K, scale=K ** -0.5)
    pos_offset = 19850
    pos = torch.arange(pos_offset + M, dtype=torch.float32)
    inv = 1.0 / (500000.0 ** (torch.arange(0, hd, 2, dtype=torch.float32) / hd))
    ang = pos[:, None] * inv[None, :]
    table = torch.stack([torch.cos(ang), torch.sin(ang)], dim=-1).contiguous().cuda()
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    rope_cols = (nq + nkv) * hd
    _gemm(A, B, out, epi=_lib.EPI_QKV_ROPE, rope=table, pos_offset=pos_offset, rope_cols=rope_cols)
    y = (A.float() @ B.float().T).view(M, -1, hd)
    c = table[pos_offset:pos_offset + M, :, 0][:, None, :]
    s = table[pos_offset:pos_offset + M, :, 1][:, None, :]
    x1, x2 = y[..., :64], y[..., 64:]
    rot = torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)
    ref = torch.cat([rot[:, :rope_cols // hd], y[:, rope_cols // hd:]], dim=1).reshape(M, N)
    assert _rel(out, ref) < TOL_BF16


# ---- short launches (M <= 256): swap-AB pair kernel, the weight as the MMA's M operand (csrc/gemm_swap.cu)
@pytest.mark.parametrize("M", [1, 8, 16, 17, 100, 128, 129, 160, 255, 256])
def test_swap_ab_unsplit_bf16_f32_silu(M):
    """K = 512 (8 k-blocks) never splits: the transposed epilogues store straight from TMEM."""
    torch.manual_seed(100 + M)
    K = 512
    A = _rand(M, K)
    B = _rand(1024, K, scale=K ** -0.5)
    ref = A.float() @ B.float().T
    out = torch.empty(M, 1024, dtype=torch.bfloat16, device="cuda")
    _gemm(A, B, out)
    assert _rel(out, ref) < TOL_BF16
    out32 = torch.empty(M, 1024, dtype=torch.float32, device="cuda")
    _gemm(A, B, out32, epi=_lib.EPI_F32)
    assert _rel(out32, ref) < TOL_F32
    I = 512
    gate, up = _rand(I, K, scale=K ** -0.5), _rand(I, K, scale=K ** -0.5)
    W = torch.stack([gate.view(I // 16, 16, K), up.view(I // 16, 16, K)], dim=1).reshape(2 * I, K).contiguous()
    act = torch.empty(M, I, dtype=torch.bfloat16, device="cuda")
    _gemm(A, W, act, epi=_lib.EPI_SILU_MUL)
    g, u = A.float() @ gate.float().T, A.float() @ up.float().T
    assert _rel(act, g / (1 + torch.exp(-g)) * u) < TOL_BF16


@pytest.mark.parametrize("M", [1, 33, 160, 256])
def test_swap_ab_strided_output_rows(M):
    """Output with a leading dimension wider than N (the engine's qkv / act rows): only [:, :N] is written."""
    torch.manual_seed(7 + M)
    K = 256
    A = _rand(M, K)
    B = _rand(512, K, scale=K ** -0.5)
    big = torch.full((M, 768), 7.0, dtype=torch.bfloat16, device="cuda")
    _gemm(A, B, big[:, :512])
    assert _rel(big[:, :512], A.float() @ B.float().T) < TOL_BF16
    assert (big[:, 512:] == 7.0).all()

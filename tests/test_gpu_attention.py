"""tcgen05 causal GQA attention (po_op_attention) vs an fp32 torch reference of _attention.

Reference semantics: ps/numerics.py:132-146 (scale 1/sqrt(d), triu mask, max-subtract softmax),
generalised to GQA heads and a q_offset (cached-prefix rows act only as keys, ps/costs.py:275-277).
Tolerance: P is rounded to bf16 before the PV product and the output is bf16 (2^-8 relative each):
8e-3 relative Frobenius error. A diagonal-dominant case pins the causal boundary exactly.
"""

import ctypes

import pytest

torch = pytest.importorskip("torch")

from paper_2505_07203_b200 import _lib  # noqa: E402

pytestmark = pytest.mark.gpu
TOL = 8e-3


def _p(t):
    return ctypes.c_void_p(t.data_ptr())


def ref_attention(qkv, n_total, q_offset, hq, hkv):
    hd = 128
    x = qkv.float()
    q = x[q_offset:, : hq * hd].view(-1, hq, hd)
    k = x[:, hq * hd:(hq + hkv) * hd].view(n_total, hkv, hd)
    v = x[:, (hq + hkv) * hd:(hq + 2 * hkv) * hd].view(n_total, hkv, hd)
    g = hq // hkv
    k = k.repeat_interleave(g, dim=1)
    v = v.repeat_interleave(g, dim=1)
    s = torch.einsum("qhd,khd->hqk", q, k) / hd ** 0.5
    pos = torch.arange(q_offset, n_total, device=qkv.device)
    keys = torch.arange(n_total, device=qkv.device)
    s = s.masked_fill(keys[None, None, :] > pos[None, :, None], float("-inf"))
    p = torch.softmax(s, dim=-1)
    return torch.einsum("hqk,khd->qhd", p, v).reshape(n_total - q_offset, hq * hd)


def run(n_total, q_offset, hq, hkv, scale=1.0, seed=0):
    torch.manual_seed(seed)
    ld = (hq + 2 * hkv) * 128
    qkv = (torch.randn(n_total, ld, device="cuda") * scale).to(torch.bfloat16)
    out = torch.full((n_total - q_offset, hq * 128), float("nan"), dtype=torch.bfloat16, device="cuda")
    _lib.call("po_op_attention", _p(qkv), ld, n_total, q_offset, hq, hkv, _p(out), hq * 128, None)
    torch.cuda.synchronize()
    ref = ref_attention(qkv, n_total, q_offset, hq, hkv)
    err = ((out.float() - ref).norm() / ref.norm()).item()
    return out, ref, err


@pytest.mark.parametrize("n,hq,hkv", [(1, 2, 1), (100, 2, 1), (128, 2, 1), (129, 4, 2), (1000, 8, 2),
                                      (2048, 2, 1), (3000, 32, 8),
                                      # odd GQA groups (Qwen-2.5-32B is 40/8): query-block-pair CTAs
                                      (1, 5, 1), (300, 5, 1), (1000, 10, 2), (2600, 40, 8), (129, 3, 3)])
def test_attention_cold(n, hq, hkv):
    out, ref, err = run(n, 0, hq, hkv, seed=n)
    assert torch.isfinite(out.float()).all()
    assert err < TOL, err


@pytest.mark.parametrize("n,off", [(300, 16), (1000, 992), (2000, 1040), (4096, 4095), (1500, 128),
                                   (20000, 19840), (20000, 19000), (9000, 8850)])
@pytest.mark.parametrize("hq,hkv", [(8, 2), (10, 2)])
def test_attention_prefix_offset(n, off, hq, hkv):
    out, ref, err = run(n, off, hq, hkv, seed=n + off)
    assert torch.isfinite(out.float()).all()
    assert err < TOL, err


def test_attention_large_logits_rescale():
    # large-magnitude scores force running-max updates (the stale-max rescale path)
    out, ref, err = run(1500, 0, 4, 2, scale=4.0, seed=5)
    assert torch.isfinite(out.float()).all()
    assert err < TOL, err


def test_attention_rejects_non_integer_group():
    qkv = torch.zeros(16, 7 * 128, dtype=torch.bfloat16, device="cuda")
    out = torch.zeros(16, 3 * 128, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(_lib.PrefillOnlyError):
        _lib.call("po_op_attention", _p(qkv), 7 * 128, 16, 0, 3, 2, _p(out), 3 * 128, None)


@pytest.mark.parametrize("n,off", [(1, 0), (200, 0), (300, 176), (1000, 512)])
def test_attention_diagonal_boundary(n, off):
    """q_i = k_i = large one-hot rows: each query attends (almost) only to its own key, so the output row
    equals v_i; any off-by-one in the causal mask is an O(1) error."""
    torch.manual_seed(n)
    hq, hkv = 2, 1
    ld = (hq + 2 * hkv) * 128
    qkv = torch.zeros(n, ld, device="cuda")
    basis = torch.nn.functional.normalize(torch.randn(n, 128, device="cuda"), dim=1)
    # random unit directions: self score 40^2/sqrt(128) ~ 141, cross scores ~ 141 * N(0, 1/128)
    qkv[:, 0:128] = basis * 40.0
    qkv[:, 128:256] = basis * 40.0
    qkv[:, 256:384] = basis * 40.0
    qkv[:, 384:512] = torch.randn(n, 128, device="cuda")
    qkv = qkv.to(torch.bfloat16)
    out = torch.zeros(n - off, hq * 128, dtype=torch.bfloat16, device="cuda")
    _lib.call("po_op_attention", _p(qkv), ld, n, off, hq, hkv, _p(out), hq * 128, None)
    torch.cuda.synchronize()
    ref = ref_attention(qkv, n, off, hq, hkv)
    assert ((out.float() - ref).abs().max() / ref.abs().max()).item() < 1e-2
    v = qkv[off:, 384:512].float()
    assert ((out[:, :128].float() - v).abs().max()).item() < 0.05


def ref_attention_rows(qkv, n_total, rows, hq, hkv):
    """fp32 reference for selected query rows only (long sequences: the full score matrix would not fit)."""
    hd = 128
    x = qkv.float()
    k = x[:, hq * hd:(hq + hkv) * hd].view(n_total, hkv, hd).repeat_interleave(hq // hkv, dim=1)
    v = x[:, (hq + hkv) * hd:(hq + 2 * hkv) * hd].view(n_total, hkv, hd).repeat_interleave(hq // hkv, dim=1)
    outs = []
    for r in rows:
        q = x[r, : hq * hd].view(hq, hd)
        s = torch.einsum("hd,khd->hk", q, k[: r + 1]) / hd ** 0.5
        outs.append(torch.einsum("hk,khd->hd", torch.softmax(s, dim=-1), v[: r + 1]).reshape(-1))
    return torch.stack(outs)


def test_attention_long_kv_banded_order():
    """12,288 keys x 8 kv heads (50 MB of K/V) switch the CTA order to kv-head bands (all heads' K/V exceed the L2
    budget); spot-check query rows across the sequence and every head."""
    n, hq, hkv = 12288, 16, 8
    torch.manual_seed(5)
    ld = (hq + 2 * hkv) * 128
    qkv = torch.randn(n, ld, device="cuda").to(torch.bfloat16)
    out = torch.full((n, hq * 128), float("nan"), dtype=torch.bfloat16, device="cuda")
    _lib.call("po_op_attention", _p(qkv), ld, n, 0, hq, hkv, _p(out), hq * 128, None)
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    rows = [0, 1, 127, 128, 4095, 6000, 9999, 12160, n - 1]
    ref = ref_attention_rows(qkv, n, rows, hq, hkv)
    got = out[rows].float()
    err = ((got - ref).norm() / ref.norm()).item()
    assert err < TOL, err


# short query suffixes over long keys: split-KV launches (packed GQA slots, head pairs, odd groups)
SPLIT_CASES = [(20000, 19840, 32, 8), (3000, 2900, 32, 8), (4000, 3424, 32, 8), (5000, 4800, 40, 8),
               (4096, 3968, 8, 2)]


@pytest.mark.parametrize("n,off,hq,hkv", SPLIT_CASES)
def test_split_kv_against_reference(n, off, hq, hkv):
    out, ref, err = run(n, off, hq, hkv, seed=off)
    assert torch.isfinite(out.float()).all()
    assert err < TOL, err
    again, _, _ = run(n, off, hq, hkv, seed=off)  # deterministic across launches
    assert torch.equal(out, again)


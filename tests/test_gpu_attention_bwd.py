"""Attention backward vs torch autograd in fp32: S <= 128 (rs_attention_bwd) and the
blocked 128 < S <= 512 kernels (rs_attention_bwd_long)."""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("B,S,H", [(1, 128, 1), (3, 64, 12), (2, 100, 4), (5, 128, 12)])
def test_attention_bwd_matches_autograd(B, S, H):
    from paper_2408_15792_b200 import _lib
    _lib.device()
    g = torch.Generator(device="cuda").manual_seed(B * S + H)
    qkv = (torch.randn(B * S, 3 * H * 64, device="cuda", generator=g)).bfloat16()
    dout = torch.randn(B * S, H * 64, device="cuda", generator=g).bfloat16()
    att = torch.empty(B * S, H * 64, dtype=torch.bfloat16, device="cuda")
    lib = _lib.load()
    _lib.check(lib.rs_attention_fwd(qkv.data_ptr(), att.data_ptr(), B, S, H, _lib.stream_handle()))
    dqkv = torch.full((B * S, 3 * H * 64), float("nan"), dtype=torch.bfloat16, device="cuda")
    _lib.check(lib.rs_attention_bwd(qkv.data_ptr(), att.data_ptr(), dout.data_ptr(), dqkv.data_ptr(), B, S, H,
                                    _lib.stream_handle()))
    x = qkv.float().requires_grad_(True)
    q, k, v = x.view(B, S, 3, H, 64).permute(2, 0, 3, 1, 4)
    o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)
    o.permute(0, 2, 1, 3).reshape(B * S, H * 64).backward(dout.float())
    ref = x.grad
    err = (dqkv.float() - ref).abs().max().item()
    scale = ref.abs().max().item()
    assert err <= 3e-2 * max(1.0, scale), (err, scale)


@pytest.mark.parametrize("B,S,H", [(1, 128, 1), (3, 64, 12), (2, 100, 4), (5, 128, 12), (2, 33, 3)])
def test_attention_bwd_lse_matches_autograd(B, S, H):
    """The training pair: the forward writes each row's log2-sum-exp, the backward takes P
    from it in one pass (two warps per row)."""
    from paper_2408_15792_b200 import _lib
    _lib.device()
    g = torch.Generator(device="cuda").manual_seed(B * S + H + 3)
    qkv = (torch.randn(B * S, 3 * H * 64, device="cuda", generator=g)).bfloat16()
    dout = torch.randn(B * S, H * 64, device="cuda", generator=g).bfloat16()
    att = torch.empty(B * S, H * 64, dtype=torch.bfloat16, device="cuda")
    lse = torch.full((B * H * S,), float("nan"), dtype=torch.float32, device="cuda")
    lib = _lib.load()
    _lib.check(lib.rs_attention_fwd_lse(qkv.data_ptr(), att.data_ptr(), lse.data_ptr(), B, S, H, _lib.stream_handle()))
    att_plain = torch.empty_like(att)
    _lib.check(lib.rs_attention_fwd(qkv.data_ptr(), att_plain.data_ptr(), B, S, H, _lib.stream_handle()))
    assert torch.equal(att, att_plain)  # the lse output changes nothing else
    x = qkv.float()
    q, k, v = x.view(B, S, 3, H, 64).permute(2, 0, 3, 1, 4)
    s = (q @ k.transpose(-1, -2)) * (0.125 * 1.4426950408889634)
    s = s.masked_fill(torch.ones(S, S, dtype=torch.bool, device="cuda").triu(1), float("-inf"))
    ref_lse = torch.logsumexp(s * 0.6931471805599453, -1) * 1.4426950408889634  # [B, H, S], log2 units
    assert torch.allclose(lse.view(B, H, S), ref_lse, atol=1e-3, rtol=1e-4)
    dqkv = torch.full((B * S, 3 * H * 64), float("nan"), dtype=torch.bfloat16, device="cuda")
    _lib.check(lib.rs_attention_bwd_lse(qkv.data_ptr(), att.data_ptr(), dout.data_ptr(), lse.data_ptr(),
                                        dqkv.data_ptr(), B, S, H, _lib.stream_handle()))
    x = qkv.float().requires_grad_(True)
    q, k, v = x.view(B, S, 3, H, 64).permute(2, 0, 3, 1, 4)
    o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)
    o.permute(0, 2, 1, 3).reshape(B * S, H * 64).backward(dout.float())
    ref = x.grad
    assert torch.isfinite(dqkv.float()).all()
    err = (dqkv.float() - ref).abs().max().item()
    scale = ref.abs().max().item()
    assert err <= 3e-2 * max(1.0, scale), (err, scale)


@pytest.mark.parametrize("fwd_lse", [False, True])
@pytest.mark.parametrize("B,S,H", [(2, 512, 4), (1, 300, 12), (3, 200, 2), (1, 129, 1), (4, 256, 12)])
def test_attention_bwd_long_matches_autograd(B, S, H, fwd_lse):
    """fwd_lse: the training path — the forward writes each row's LSE and the dQ kernel
    takes it instead of recomputing the row statistics (rs_attention_bwd_long_lse)."""
    from paper_2408_15792_b200 import _lib
    _lib.device()
    g = torch.Generator(device="cuda").manual_seed(B * S + H + 7)
    qkv = (torch.randn(B * S, 3 * H * 64, device="cuda", generator=g)).bfloat16()
    dout = torch.randn(B * S, H * 64, device="cuda", generator=g).bfloat16()
    att = torch.empty(B * S, H * 64, dtype=torch.bfloat16, device="cuda")
    lib = _lib.load()
    lse = torch.full((B * H * S,), float("nan"), dtype=torch.float32, device="cuda")
    _lib.check(lib.rs_attention_fwd_lse(qkv.data_ptr(), att.data_ptr(), lse.data_ptr(), B, S, H, _lib.stream_handle()))
    dqkv = torch.full((B * S, 3 * H * 64), float("nan"), dtype=torch.bfloat16, device="cuda")
    n_ws = lib.rs_attention_bwd_long_workspace_size(B, S, H)
    ws = torch.full((n_ws,), 0xFF, dtype=torch.uint8, device="cuda")  # NaN scratch: must be written before read
    if fwd_lse:
        _lib.check(lib.rs_attention_bwd_long_lse(qkv.data_ptr(), att.data_ptr(), dout.data_ptr(), lse.data_ptr(),
                                                 dqkv.data_ptr(), B, S, H, ws.data_ptr(), n_ws, _lib.stream_handle()),
                   "rs_attention_bwd_long_lse")
    else:
        _lib.check(lib.rs_attention_bwd_long(qkv.data_ptr(), att.data_ptr(), dout.data_ptr(), dqkv.data_ptr(), B, S,
                                             H, ws.data_ptr(), n_ws, _lib.stream_handle()), "rs_attention_bwd_long")
    x = qkv.float().requires_grad_(True)
    q, k, v = x.view(B, S, 3, H, 64).permute(2, 0, 3, 1, 4)
    o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)
    o.permute(0, 2, 1, 3).reshape(B * S, H * 64).backward(dout.float())
    ref = x.grad
    assert torch.isfinite(dqkv.float()).all()
    err = (dqkv.float() - ref).abs().max().item()
    scale = ref.abs().max().item()
    assert err <= 3e-2 * max(1.0, scale), (err, scale)
    rel = ((dqkv.float() - ref).norm() / ref.norm()).item()
    assert rel <= 1e-2, rel


def test_attention_bwd_long_rejects_out_of_range():
    from paper_2408_15792_b200 import _lib
    _lib.device()
    lib = _lib.load()
    assert lib.rs_attention_bwd_long(None, None, None, None, 1, 513, 1, None, 0, None) == _lib.RS_ERR_INVALID

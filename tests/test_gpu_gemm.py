"""K3 tcgen05 GEMM with fused epilogues vs a plain fp32 torch reference."""

import ctypes

import pytest
import torch

pytestmark = pytest.mark.gpu


def _gemm(A, W, bias, R, epi):
    from paper_2408_15792_b200 import _lib
    _lib.device()
    M, K = A.shape
    N = W.shape[0]
    C = torch.empty(M, N, dtype=torch.float32 if epi == 2 else torch.bfloat16, device=A.device)
    _lib.check(_lib.load().rs_gemm_bf16(A.data_ptr(), W.data_ptr(), bias.data_ptr(),
                                        None if R is None else R.data_ptr(), C.data_ptr(), M, N, K, epi,
                                        _lib.stream_handle()))
    return C


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 768, 768), (1024, 2304, 768), (512, 3072, 768),
                                   (384, 768, 3072), (128 * 300, 768, 768)])
@pytest.mark.parametrize("epi", [0, 1, 2, 3])
def test_gemm_matches_fp32(M, N, K, epi):
    g = torch.Generator(device="cuda").manual_seed(M + N + K + epi)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.05).bfloat16()
    bias = torch.randn(N, device="cuda", generator=g).bfloat16()
    R = torch.randn(M, N, device="cuda", generator=g) if epi == 2 else None
    C = _gemm(A, W, bias, R, epi).float()
    ref = A.float() @ W.float().t() + bias.float()
    if epi == 1:
        ref = torch.relu(ref)
    elif epi == 2:
        ref = ref + R
    elif epi == 3:
        ref = torch.nn.functional.gelu(ref, approximate="tanh")
    err = (C - ref).abs().max().item()
    tol = 2e-2 * max(1.0, ref.abs().max().item())
    assert err <= tol, (err, tol)


def test_gemm_rejects_bad_shapes():
    from paper_2408_15792_b200 import _lib
    _lib.device()
    A = torch.zeros(100, 64, dtype=torch.bfloat16, device="cuda")
    W = torch.zeros(256, 64, dtype=torch.bfloat16, device="cuda")
    b = torch.zeros(256, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError):
        _gemm(A, W, b, None, 0)


def test_gemm_residual_in_place():
    g = torch.Generator(device="cuda").manual_seed(7)
    A = torch.randn(256, 768, device="cuda", generator=g).bfloat16()
    W = (torch.randn(768, 768, device="cuda", generator=g) * 0.05).bfloat16()
    b = torch.randn(768, device="cuda", generator=g).bfloat16()
    h = torch.randn(256, 768, device="cuda", generator=g)
    want = h + A.float() @ W.float().t() + b.float()
    from paper_2408_15792_b200 import _lib
    _lib.check(_lib.load().rs_gemm_bf16(A.data_ptr(), W.data_ptr(), b.data_ptr(), h.data_ptr(), h.data_ptr(),
                                        256, 768, 768, 2, _lib.stream_handle()))
    assert (h - want).abs().max().item() < 1e-3

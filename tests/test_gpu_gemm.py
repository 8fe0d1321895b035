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


def _gemm_ex(A, W, aux, M, N, K, epi, a_mn, b_mn, splits=1, bias=None, out_dtype=torch.float32):
    from paper_2408_15792_b200 import _lib
    _lib.device()
    rows = M * (splits if epi == 6 else 1)
    C = torch.empty(rows, N, dtype=out_dtype, device="cuda")
    _lib.check(_lib.load().rs_gemm_bf16_ex(A.data_ptr(), W.data_ptr(), None if bias is None else bias.data_ptr(),
                                           None if aux is None else aux.data_ptr(), C.data_ptr(), M, N, K, epi,
                                           a_mn, b_mn, splits, _lib.stream_handle()))
    return C


@pytest.mark.parametrize("T,Nf,Kin", [(512, 768, 3072), (1024, 3072, 768), (256, 2304, 768), (768, 768, 768)])
def test_dgrad_matches_fp32(T, Nf, Kin):
    """dX[T, Kin] = dY[T, Nf] . W[Nf, Kin] with W read MN-major (the backward data GEMM)."""
    g = torch.Generator(device="cuda").manual_seed(T + Nf)
    dY = torch.randn(T, Nf, device="cuda", generator=g).bfloat16()
    W = (torch.randn(Nf, Kin, device="cuda", generator=g) * 0.05).bfloat16()
    ref = dY.float() @ W.float()
    C = _gemm_ex(dY, W, None, T, Kin, Nf, 4, 0, 1)
    assert (C - ref).abs().max().item() <= 2e-2 * max(1.0, ref.abs().max().item())
    mask = torch.randn(T, Kin, device="cuda", generator=g).bfloat16()
    Cm = _gemm_ex(dY, W, mask, T, Kin, Nf, 5, 0, 1, out_dtype=torch.bfloat16).float()
    refm = ref * (mask.float() > 0)
    assert (Cm - refm).abs().max().item() <= 2e-2 * max(1.0, ref.abs().max().item())


@pytest.mark.parametrize("T,Nf,Kin,splits", [(4096, 768, 3072, 1), (8192, 3072, 768, 4), (2048, 768, 768, 8),
                                             (1024, 2304, 768, 3)])
def test_wgrad_matches_fp32(T, Nf, Kin, splits):
    """dW[Nf, Kin] = dY^T X over T tokens: both operands MN-major; split-K partial slices."""
    g = torch.Generator(device="cuda").manual_seed(T + Kin)
    dY = torch.randn(T, Nf, device="cuda", generator=g).bfloat16()
    X = torch.randn(T, Kin, device="cuda", generator=g).bfloat16()
    ref = dY.float().t() @ X.float()
    epi = 6 if splits > 1 else 4
    C = _gemm_ex(dY, X, None, Nf, Kin, T, epi, 1, 1, splits)
    got = C.view(splits, Nf, Kin).sum(0) if splits > 1 else C
    assert (got - ref).abs().max().item() <= 1e-2 * max(1.0, ref.abs().max().item())


def test_gemm_qkv_f16_v_epilogue():
    """Epilogue 7: bf16 q|k columns, fp16 v columns (the last third)."""
    from paper_2408_15792_b200 import _lib
    _lib.device()
    M, N, K = 512, 2304, 768
    g = torch.Generator(device="cuda").manual_seed(3)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.05).bfloat16()
    b = (torch.randn(N, device="cuda", generator=g) * 0.1).bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    _lib.check(_lib.load().rs_gemm_bf16(A.data_ptr(), W.data_ptr(), b.data_ptr(), None, C.data_ptr(), M, N, K, 7,
                                        _lib.stream_handle()))
    ref = A.float() @ W.float().t() + b.float()
    qk = C[:, :2 * N // 3].float()
    v = C[:, 2 * N // 3:].view(torch.float16).float()
    torch.testing.assert_close(qk, ref[:, :2 * N // 3], rtol=2e-2, atol=2e-2)
    torch.testing.assert_close(v, ref[:, 2 * N // 3:], rtol=2e-3, atol=2e-3)

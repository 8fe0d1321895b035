"""Time the four OPT projection GEMMs at M = 2^20 (CUDA events, 10 reps)."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2408_15792_b200 import _lib
_lib.device()
lib = _lib.load()
M = 1 << 20
for N, K, epi in [(2304, 768, 0), (768, 768, 2), (3072, 768, 1), (768, 3072, 2)]:
    A = torch.randn(M, K, device="cuda").bfloat16()
    W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
    b = torch.zeros(N, device="cuda").bfloat16()
    C = torch.randn(M, N, device="cuda", dtype=torch.float32 if epi == 2 else torch.bfloat16)
    f = lambda: _lib.check(lib.rs_gemm_bf16(A.data_ptr(), W.data_ptr(), b.data_ptr(), C.data_ptr() if epi == 2 else None,
                                            C.data_ptr(), M, N, K, epi, _lib.stream_handle()))
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): f()
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10
    print(f"gemm N={N} K={K} epi={epi}: {t:.3f} ms {2*M*N*K/t/1e9:.0f} TFLOP/s", flush=True)
    del A, W, C

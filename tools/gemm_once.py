"""Launch one GEMM (for ncu captures): python tools/gemm_once.py M N K epi [reps]"""
import sys
import pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2408_15792_b200 import _lib

M, N, K, epi = (int(v) for v in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
_lib.device()
A = torch.randn(M, K, device="cuda").bfloat16()
W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
b = torch.zeros(N, device="cuda").bfloat16()
C = torch.empty(M, N, device="cuda", dtype=torch.float32 if epi == 2 else torch.bfloat16)
for _ in range(reps):
    _lib.check(_lib.load().rs_gemm_bf16(A.data_ptr(), W.data_ptr(), b.data_ptr(), C.data_ptr() if epi == 2 else None,
                                        C.data_ptr(), M, N, K, epi, _lib.stream_handle()))
torch.cuda.synchronize()
print("ok")

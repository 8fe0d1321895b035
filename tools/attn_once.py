"""Launch the attention kernel (for ncu): python tools/attn_once.py B S [reps]"""
import sys
import pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2408_15792_b200 import _lib

B, S = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
_lib.device()
qkv = torch.randn(B * S, 2304, device="cuda").bfloat16()
out = torch.empty(B * S, 768, device="cuda").bfloat16()
for _ in range(reps):
    _lib.check(_lib.load().rs_attention_fwd_f16v(qkv.data_ptr(), out.data_ptr(), B, S, 12, _lib.stream_handle()))
torch.cuda.synchronize()
print("ok")

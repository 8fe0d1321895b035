import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2408_15792_b200 import _lib
_lib.device()
B = 2048
qkv = (torch.randn(B * 512, 2304, device="cuda") * 0.5).bfloat16(); out = torch.empty(B * 512, 768, device="cuda").bfloat16()
tr = torch.zeros(64 * 8, dtype=torch.int64, device="cuda")
for _ in range(2):
    tr.zero_()
    _lib.check(_lib.load().rs_attention_fwd_trace(qkv.data_ptr(), out.data_ptr(), B, 512, 12, tr.data_ptr(), _lib.stream_handle()))
torch.cuda.synchronize()
t = tr.view(64, 8).cpu().numpy()
base = t[0, 0]
names = ["start", "s_full", "barmax", "p_empty", "stored", "pre_ofull", "o_full", "o_done"]
for i in range(40):
    row = t[i]
    print(i, " ".join(f"{n}={(v - base) if v else '-':>8}" for n, v in zip(names, row)))

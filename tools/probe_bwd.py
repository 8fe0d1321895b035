"""Run attention fwd / bwd for one shape (argv: which B S H); print max error vs torch."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2408_15792_b200 import _lib

which, B, S, H = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
_lib.device()
lib = _lib.load()
g = torch.Generator(device="cuda").manual_seed(B * S + H)
qkv = torch.randn(B * S, 3 * H * 64, device="cuda", generator=g).bfloat16()
dout = torch.randn(B * S, H * 64, device="cuda", generator=g).bfloat16()
att = torch.empty(B * S, H * 64, dtype=torch.bfloat16, device="cuda")
_lib.check(lib.rs_attention_fwd(qkv.data_ptr(), att.data_ptr(), B, S, H, _lib.stream_handle()))
torch.cuda.synchronize()
x = qkv.float().requires_grad_(True)
q, k, v = x.view(B, S, 3, H, 64).permute(2, 0, 3, 1, 4)
o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)
o = o.permute(0, 2, 1, 3).reshape(B * S, H * 64)
print("fwd err", (att.float() - o).abs().max().item(), flush=True)
if which == "bwd":
    dqkv = torch.zeros(B * S, 3 * H * 64, dtype=torch.bfloat16, device="cuda")
    _lib.check(lib.rs_attention_bwd(qkv.data_ptr(), att.data_ptr(), dout.data_ptr(), dqkv.data_ptr(), B, S, H,
                                    _lib.stream_handle()))
    torch.cuda.synchronize()
    o.backward(dout.float())
    ref = x.grad
    d = (dqkv.float() - ref).abs()
    print("bwd err", d.max().item(), "scale", ref.abs().max().item(), "per-part",
          [d.view(B * S, 3, H * 64)[:, i].max().item() for i in range(3)], flush=True)

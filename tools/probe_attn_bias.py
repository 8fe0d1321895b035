"""Attention forward error statistics vs fp32 (bias / RMS), bf16 and fp16-V paths."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2408_15792_b200 import _lib
_lib.device()
lib = _lib.load()
for (B, S, H, scale) in [(24, 128, 4, 0.3), (24, 128, 4, 1.5), (8, 512, 12, 0.3), (8, 512, 12, 1.5), (16, 100, 4, 0.5)]:
    g = torch.Generator(device="cuda").manual_seed(B * S + H)
    x = torch.randn(B * S, 3 * H * 64, device="cuda", generator=g) * scale
    d = H * 64
    for f16v in (0, 1):
        qkv = x.bfloat16()
        if f16v:
            qkv[:, 2 * d:] = x[:, 2 * d:].half().view(torch.bfloat16)
            ref_in = torch.cat([qkv[:, :2 * d].float(), qkv[:, 2 * d:].view(torch.float16).float()], 1)
            fn = lib.rs_attention_fwd_f16v
        else:
            ref_in = qkv.float()
            fn = lib.rs_attention_fwd
        out = torch.empty(B * S, d, dtype=torch.bfloat16, device="cuda")
        _lib.check(fn(qkv.data_ptr(), out.data_ptr(), B, S, H, _lib.stream_handle()))
        q, k, v = ref_in.view(B, S, 3, H, 64).permute(2, 0, 3, 1, 4)
        ref = torch.nn.functional.scaled_dot_product_attention(q.double(), k.double(), v.double(), is_causal=True)
        ref = ref.permute(0, 2, 1, 3).reshape(B * S, d)
        err = out.double() - ref
        rb = ref.bfloat16().double() - ref  # bf16 output rounding alone
        print(f"B={B} S={S} H={H} scale={scale} f16v={f16v}: max {err.abs().max():.2e} rms {err.pow(2).mean().sqrt():.2e} "
              f"mean {err.mean():+.2e} | bf16-rounding rms {rb.pow(2).mean().sqrt():.2e} mean {rb.mean():+.2e} "
              f"| ref rms {ref.pow(2).mean().sqrt():.2e}", flush=True)

"""Timeline of attention CTA 0 (diagnostics): softmax phases per block and MMA issue."""
import sys, pathlib, ctypes
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2408_15792_b200 import _lib
_lib.device()
lib = _lib.load()
fn = lib.rs_attention_fwd_trace
fn.restype = ctypes.c_int
fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p,
               ctypes.c_void_p]
B = 2048
qkv = (torch.randn(B * 512, 2304, device="cuda") * 0.5).bfloat16()
out = torch.empty(B * 512, 768, device="cuda").bfloat16()
tr = torch.zeros(8192, dtype=torch.int64, device="cuda")
for _ in range(2):
    tr.zero_()
    _lib.check(fn(qkv.data_ptr(), out.data_ptr(), B, 512, 12, tr.data_ptr(), _lib.stream_handle()))
torch.cuda.synchronize()
t = tr.cpu().numpy()
base = min(v for v in t if v > 0)
sm = t[:512].reshape(2, 64, 4)
mm = t[1024:1280].reshape(2, 64, 2)
cc = t[2048:2560].reshape(2, 64, 4)
si = t[3072:3584].reshape(2, 64, 4)
pv = t[4096:4608].reshape(2, 64, 4)
oc = t[5120:5376].reshape(2, 64, 2)
ev = []
for s in range(2):
    for b in range(40):
        w0, sf, p1, p2 = sm[s, b]
        if sf:
            c0, c1, c2, c3 = cc[s, b]
            ev.append((sf - base, f"slot{s} blk{b:2d}: wait {sf - w0:5d}  pass1 {p1 - sf:5d}  pass2 {p2 - p1:5d}"
                                  f"  [chunk1: ld {c1 - c0:4d} exp {c2 - c1:4d} st {c3 - c2:4d}]"))
        ms, me = mm[s, b]
        if ms:
            a, q, kv, e = si[s, b + 1] if b + 1 < 64 else (0, 0, 0, 0)
            ev.append((ms - base, f"   MMA slot{s} blk{b:2d}: p_full seen, issue took {me - ms:4d}"
                                  f"  [pre {pv[s,b,0] - ms:5d} mma {pv[s,b,1] - pv[s,b,0]:5d} post {pv[s,b,2] - pv[s,b,1]:5d}"
                                  f" (kvc {pv[s,b,3] - pv[s,b,1]:5d} oc {(oc[s,b,0] - pv[s,b,3]) if oc[s,b,0] else 0:5d})"
                                  f" q {q - a:5d} kv {kv - q:5d} S {e - kv:5d}]"))
for when, txt in sorted(ev)[:120]:
    print(f"{when:8d} {txt}")

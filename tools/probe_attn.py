import sys, pathlib, subprocess, threading, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2408_15792_b200 import _lib
_lib.device()
def clk():
    return subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for B in (2048, 512):
    qkv = (torch.randn(B * 512, 2304, device="cuda") * 0.5).bfloat16(); out = torch.empty(B * 512, 768, device="cuda").bfloat16()
    f = lambda: _lib.load().rs_attention_fwd_f16v(qkv.data_ptr(), out.data_ptr(), B, 512, 12, _lib.stream_handle())
    f(); torch.cuda.synchronize()
    for reps in (1, 3, 10):
        e0.record()
        for _ in range(reps): f()
        e1.record(); torch.cuda.synchronize(); t = e0.elapsed_time(e1)/reps
        print(f"attention B={B} reps={reps}: {t:.3f} ms {2*768*512*513*B/t/1e9:.0f} TFLOP/s  clk {clk()}", flush=True)

import time, torch, sys
sys.path.insert(0, '.')
from paper_2408_15792_b200.ranker import OptRanker, RankerConfig
from paper_2408_15792_b200 import _lib
cfg = RankerConfig.opt_125m()
m = OptRanker(cfg, seed=0)
B, S = 4096, 512
ids = torch.randint(4, cfg.vocab, (B, S), dtype=torch.int32, device="cuda")
for _ in range(2): m.forward(ids)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); 
for _ in range(3): m.forward(ids)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
fl = cfg.flops_per_prompt(S) * B
print(f"forward {B}x{S}: {ms:.1f} ms  {B/ms*1e3:.0f} prompts/s  {fl/ms/1e9:.1f} TFLOP/s")
# per-kernel timings
M = 1 << 20
def tg(N, K, epi, n=10):
    A = torch.randn(M, K, device="cuda").bfloat16(); W = torch.randn(N, K, device="cuda").bfloat16()*0.02
    b = torch.zeros(N, device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.float32 if epi == 2 else torch.bfloat16)
    R = torch.zeros(M, N, device="cuda") if epi == 2 else None
    f = lambda: _lib.load().rs_gemm_bf16(A.data_ptr(), W.data_ptr(), b.data_ptr(), None if R is None else R.data_ptr(), C.data_ptr(), M, N, K, epi, _lib.stream_handle())
    f(); torch.cuda.synchronize(); e0.record()
    for _ in range(n): f()
    e1.record(); torch.cuda.synchronize(); t = e0.elapsed_time(e1)/n
    print(f"gemm M={M} N={N} K={K} epi={epi}: {t:.3f} ms {2*M*N*K/t/1e9:.0f} TFLOP/s")
tg(2304, 768, 0); tg(768, 768, 2); tg(3072, 768, 1); tg(768, 3072, 2)
qkv = torch.randn(2048*512, 2304, device="cuda").bfloat16(); out = torch.empty(2048*512, 768, device="cuda").bfloat16()
f = lambda: _lib.load().rs_attention_fwd(qkv.data_ptr(), out.data_ptr(), 2048, 512, 12, _lib.stream_handle())
f(); torch.cuda.synchronize(); e0.record()
for _ in range(5): f()
e1.record(); torch.cuda.synchronize(); t = e0.elapsed_time(e1)/5
afl = 2*768*512*513*2048
print(f"attention 2048x512: {t:.3f} ms {afl/t/1e9:.0f} TFLOP/s")
import subprocess
print(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active", "--format=csv"], capture_output=True, text=True).stdout)

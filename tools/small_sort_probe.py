"""Rank step at small queue sizes: one-CTA bitonic sort (default) vs the block-sort merge
path (RSB200_LIB=variants/librsb200_nosmall.so). Prints ms per step (eager, CUDA events)."""
import pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2408_15792_b200 import _lib
from paper_2408_15792_b200.schedulers import DeviceQueue, SchedulerConfig
_lib.device()
cfg = SchedulerConfig(max_batch=256, starvation_threshold=100, priority_quantum=50)
g = torch.Generator(device="cuda").manual_seed(0)
for n in (300, 600, 1000, 1500, 2000):
    dq = DeviceQueue(n, torch.device("cuda"), score_dtype=torch.float64)
    dq.score.copy_(torch.randn(n, device="cuda", generator=g, dtype=torch.float64))
    dq.flags.fill_(_lib.RS_FLAG_SCORED)
    dq.arrival_rank.copy_(torch.arange(n, dtype=torch.int32))
    for _ in range(3):
        dq.rank_step(cfg, None, length_calibrated=False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(50):
        dq.rank_step(cfg, None, length_calibrated=False)
    e1.record(); torch.cuda.synchronize()
    print(n, f"{e0.elapsed_time(e1) / 50 * 1000:.1f} us")

"""Profiling driver: the tau fast path and the rank step at a given size (for ncu).
usage: python tools/prof_sort.py [tau|rank] N [reps]"""
import sys
import pathlib

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    what, n = sys.argv[1], int(sys.argv[2])
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    g = torch.Generator(device="cuda").manual_seed(11)
    if what == "tau":
        from paper_2408_15792_b200 import ranking
        x = torch.randn(n, device="cuda", generator=g)
        y = torch.randint(1, 2049, (n,), device="cuda", generator=g, dtype=torch.int32)
        out = torch.empty(6, dtype=torch.int64, device="cuda")
        for _ in range(reps):
            ranking.tau_counts_device(x, y, out, fast_only=True)
        torch.cuda.synchronize()
        print("tau", out.tolist())
    else:
        from paper_2408_15792_b200 import _lib
        from paper_2408_15792_b200.schedulers import DeviceQueue, SchedulerConfig
        dq = DeviceQueue(n, torch.device("cuda"), score_dtype=torch.float32)
        dq.score.copy_(torch.randn(n, device="cuda", generator=g))
        dq.flags.fill_(_lib.RS_FLAG_SCORED)
        dq.arrival_rank.copy_(torch.arange(n, dtype=torch.int32))
        cfg = SchedulerConfig(max_batch=256, starvation_threshold=100, priority_quantum=50)
        for _ in range(reps):
            dq.rank_step(cfg, None, length_calibrated=False)
        torch.cuda.synchronize()
        print("rank ok")


if __name__ == "__main__":
    main()

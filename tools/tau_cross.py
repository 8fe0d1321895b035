"""Crossover of the two exact tau paths (RS_TAU_PATH=general|fast), device time per call
(CUDA events, 5 calls after a warm-up) on cfg4-shaped inputs (x N(0,1) f32, y U[1, 2048])."""
import os
import pathlib
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2408_15792_b200 import ranking  # noqa: E402


def main():
    g = torch.Generator(device="cuda").manual_seed(3)
    for lg in range(16, 27):
        n = 1 << lg
        x = torch.randn(n, device="cuda", generator=g)
        y = torch.randint(1, 2049, (n,), device="cuda", generator=g, dtype=torch.int32)
        out = torch.empty(6, dtype=torch.int64, device="cuda")
        row = [n]
        for path in ("general", "fast"):
            os.environ["RS_TAU_PATH"] = path
            ranking.tau_counts_device(x, y, out, fast_only=True)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                ranking.tau_counts_device(x, y, out, fast_only=True)
            e1.record()
            torch.cuda.synchronize()
            row.append(e0.elapsed_time(e1) / 5)
        os.environ.pop("RS_TAU_PATH")
        plan = ranking.TauPlan(x, y)
        plan()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            plan()
        e1.record()
        torch.cuda.synchronize()
        row.append(e0.elapsed_time(e1) / 5)
        print(f"n=2^{lg}: general {row[1]:.3f} ms  fast {row[2]:.3f} ms  default-path graph {row[3]:.3f} ms",
              flush=True)
        del plan


if __name__ == "__main__":
    main()

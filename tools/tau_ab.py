"""Tau fast path vs general path (exact counts must agree) on assorted inputs, then the
fast path's timing by size (CUDA events) and the cfg4 1M recipe as a graph."""
import os
import pathlib
import sys
ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))
import torch  # noqa: E402
from paper_2408_15792_b200 import ranking  # noqa: E402


def counts(x, y, path):
    os.environ["RS_TAU_PATH"] = path
    r = ranking.tau_counts_device(x, y).cpu().tolist()
    os.environ.pop("RS_TAU_PATH")
    return r


g = torch.Generator(device="cuda").manual_seed(3)
bad = 0
cases = []
for n in (1, 2, 100, 1000, 5000, 70000, 1 << 18, 1 << 20, 3 << 20, 1 << 24):
    cases.append((f"randn/len n={n}", torch.randn(n, device="cuda", generator=g),
                  torch.randint(1, 2049, (n,), device="cuda", generator=g, dtype=torch.int32)))
for n in (1000, 1 << 20):
    cases.append((f"rounded x (ties) n={n}", (torch.randn(n, device="cuda", generator=g) * 8).round(),
                  torch.randint(0, 40, (n,), device="cuda", generator=g, dtype=torch.int32)))
    cases.append((f"uniform x n={n}", torch.rand(n, device="cuda", generator=g),
                  torch.randint(0, 4000, (n,), device="cuda", generator=g, dtype=torch.int32)))
    y = torch.randint(1, 2049, (n,), device="cuda", generator=g, dtype=torch.int32)
    cases.append((f"x = y + noise n={n}", y.float() + torch.randn(n, device="cuda", generator=g), y))
    cases.append((f"int x few values n={n}", torch.randint(0, 5000, (n,), device="cuda", generator=g,
                                                           dtype=torch.int32).float(), y))
    cases.append((f"heavy tails n={n}", torch.randn(n, device="cuda", generator=g) ** 5, y))
if "--time-only" not in sys.argv:
    for name, x, y in cases:
        a, b = counts(x, y, "fast"), counts(x, y, "general")
        ok = a[:5] == b[:5]
        bad += not ok
        print(("ok  " if ok else "BAD ") + name, a if not ok else "", b if not ok else "", flush=True)
    print("mismatches", bad)


if "--check-only" in sys.argv:
    sys.exit(1 if bad else 0)


def timed(fn, reps=10):
    fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


res = torch.empty(6, dtype=torch.int64, device="cuda")
for n in (1 << 18, 1 << 20, 1 << 24, 1 << 26, 1 << 28):
    x = torch.randn(n, device="cuda", generator=g)
    y = torch.randint(1, 2049, (n,), device="cuda", generator=g, dtype=torch.int32)
    t = timed(lambda: ranking.tau_counts_device(x, y, res, fast_only=True), 3 if n >= 1 << 26 else 10)
    os.environ["RS_TAU_PATH"] = "general"
    tg = timed(lambda: ranking.tau_counts_device(x, y, res), 3) if n <= 1 << 20 else float("nan")
    os.environ.pop("RS_TAU_PATH")
    print(f"n={n}: fast {t:.4f} ms  general {tg:.4f} ms  status {int(res[5])}", flush=True)
    del x, y
import recipes  # noqa: E402
xn, yn = recipes.tau_1m("f32")
x, y = torch.from_numpy(xn).cuda(), torch.from_numpy(yn).cuda()
plan = ranking.TauPlan(x, y)
t = timed(plan, 20)
print(f"cfg4 1M graph {t:.4f} ms", plan.counts())

"""RS_TAU_CAP sweep of the tau fast path at several sizes (and the fast / general
crossover below 2^18): python tools/tau_cap_sweep.py"""
import os
import pathlib
import sys
ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))
import torch  # noqa: E402
from paper_2408_15792_b200 import ranking  # noqa: E402


def timed(fn, reps=20):
    fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


g = torch.Generator(device="cuda").manual_seed(5)
res = torch.empty(6, dtype=torch.int64, device="cuda")
import recipes  # noqa: E402
xn, yn = recipes.tau_1m("f32")
inputs = {"cfg4-1M": (torch.from_numpy(xn).cuda(), torch.from_numpy(yn).cuda())}
for n in (1 << 16, 1 << 17, 1 << 18, 1 << 20, 1 << 22, 1 << 24):
    inputs[f"randn-{n}"] = (torch.randn(n, device="cuda", generator=g),
                            torch.randint(1, 2049, (n,), device="cuda", generator=g, dtype=torch.int32))
for name, (x, y) in inputs.items():
    row = []
    for cap in ("", "1024", "2048", "4096", "8192"):
        if cap:
            os.environ["RS_TAU_CAP"] = cap
        os.environ["RS_TAU_PATH"] = "fast"
        t = timed(lambda: ranking.tau_counts_device(x, y, res))
        os.environ.pop("RS_TAU_CAP", None)
        row.append(f"cap={cap or 'auto'}:{t:.4f}")
    os.environ["RS_TAU_PATH"] = "general"
    tg = timed(lambda: ranking.tau_counts_device(x, y, res))
    os.environ.pop("RS_TAU_PATH")
    print(name, " ".join(row), f"general:{tg:.4f}", flush=True)

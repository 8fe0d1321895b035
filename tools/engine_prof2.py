"""The cfg5 engine loop (generate_poisson(40, n, sharegpt, seed 7, noise 0.25), random
scores as the score cache, max_batch 256, starvation 100 / 50, default cost preset):
wall time per step, for ncu launch lists of a steady-state window.
usage: python tools/engine_prof2.py [n] [stop_after_finished]"""
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
from paper_2408_15792_b200 import engine  # noqa: E402
from paper_2408_15792_b200.schedulers import SchedulerConfig  # noqa: E402
from paper_2408_15792_b200.workload import LengthDist, generate_poisson  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
stop = int(sys.argv[2]) if len(sys.argv) > 2 else None
trace = generate_poisson(40.0, n, LengthDist.parse("sharegpt"), seed=7, prompt_noise=0.25)
reqs = list(trace)
scores = np.random.default_rng(8).normal(size=n)
sched = SchedulerConfig(max_batch=256, starvation_threshold=100, priority_quantum=50)
eng = engine.DeviceEngine(reqs, scores, sched, engine.COST_PRESETS["default"])
t0 = time.perf_counter()
res = eng.run(stop_after_finished=stop)
dt = time.perf_counter() - t0
print(n, res.steps, "steps", f"{dt:.2f} s", f"{dt / max(res.steps, 1) * 1e6:.1f} us/step", res.metrics["n_finished"])

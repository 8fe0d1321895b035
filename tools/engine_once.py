"""Run the device engine loop on a synthetic Poisson trace (for ncu launch lists)."""
import sys, pathlib, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2408_15792_b200 import engine
from paper_2408_15792_b200.schedulers import SchedulerConfig
import bench
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
reqs, _ = bench.synthetic_poisson(n)
scores = np.random.default_rng(8).normal(size=n)
eng = engine.DeviceEngine(reqs, scores, SchedulerConfig(max_batch=256, starvation_threshold=100, priority_quantum=50))
t0 = time.perf_counter()
res = eng.run(stop_after_finished=int(sys.argv[2]) if len(sys.argv) > 2 else None)
dt = time.perf_counter() - t0
print(n, res.steps, "steps", f"{dt:.2f} s", f"{res.steps / dt:.0f} steps/s", res.metrics["n_finished"])

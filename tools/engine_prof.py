"""cProfile of the device engine host loop + an nsys-free kernel census (ncu launch list
is separate): where a step's ~250 us go."""
import cProfile
import pathlib
import pstats
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import bench  # noqa: E402
from paper_2408_15792_b200 import engine  # noqa: E402
from paper_2408_15792_b200.schedulers import SchedulerConfig  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
reqs, _ = bench.synthetic_poisson(n)
scores = np.random.default_rng(8).normal(size=n)
cfg = SchedulerConfig(max_batch=256, starvation_threshold=100, priority_quantum=50)
eng = engine.DeviceEngine(reqs, scores, cfg)
eng.run(stop_after_finished=200)
eng = engine.DeviceEngine(reqs, scores, cfg)
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
res = eng.run()
pr.disable()
dt = time.perf_counter() - t0
print(n, res.steps, "steps", f"{dt:.2f} s", f"{dt / res.steps * 1e6:.1f} us/step")
pstats.Stats(pr).sort_stats("tottime").print_stats(18)

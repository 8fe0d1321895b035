"""The cfg5 engine loop run twice — the one-launch device loop and the per-kernel host
loop (RS_ENGINE_LOOP=host in a child process) — same rows and metrics, and each's time.
usage: python tools/engine_ab.py [n]"""
import json
import os
import pathlib
import subprocess
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
if os.environ.get("_AB_CHILD"):
    import hashlib
    import numpy as np
    from paper_2408_15792_b200 import engine
    from paper_2408_15792_b200.schedulers import SchedulerConfig
    from paper_2408_15792_b200.workload import LengthDist, generate_poisson
    reqs = list(generate_poisson(40.0, n, LengthDist.parse("sharegpt"), seed=7, prompt_noise=0.25))
    scores = np.random.default_rng(8).normal(size=n)
    sched = SchedulerConfig(max_batch=256, starvation_threshold=100, priority_quantum=50)
    eng = engine.DeviceEngine(reqs, scores, sched, engine.COST_PRESETS["default"])
    eng.run(stop_after_finished=min(n, 200))  # warm-up (fresh engine below)
    eng = engine.DeviceEngine(reqs, scores, sched, engine.COST_PRESETS["default"])
    t0 = time.perf_counter()
    res = eng.run()
    dt = time.perf_counter() - t0
    h = hashlib.sha256(json.dumps(res.requests, sort_keys=True).encode()).hexdigest()
    print(json.dumps({"s": dt, "steps": res.steps, "us_per_step": dt / max(res.steps, 1) * 1e6,
                      "rows": h, "metrics": res.metrics}))
    sys.exit(0)
out = {}
for mode in ("device", "host"):
    env = dict(os.environ, _AB_CHILD="1")
    if mode == "host":
        env["RS_ENGINE_LOOP"] = "host"
    p = subprocess.run([sys.executable, __file__, str(n)], env=env, capture_output=True, text=True, timeout=900)
    if p.returncode:
        print(mode, "FAILED", p.stderr[-2000:])
        sys.exit(1)
    out[mode] = json.loads(p.stdout.strip().splitlines()[-1])
    print(mode, "%.3f s" % out[mode]["s"], out[mode]["steps"], "steps", "%.1f us/step" % out[mode]["us_per_step"])
same = out["device"]["rows"] == out["host"]["rows"] and out["device"]["metrics"] == out["host"]["metrics"]
print("identical:", same)
sys.exit(0 if same else 2)

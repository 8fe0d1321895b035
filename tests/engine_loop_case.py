"""Helper for tests/test_gpu_engine_loop.py (not a test module): one record-free engine run
of a named configuration, printed as JSON (sha256 of the per-request rows, the metrics,
the step count). The test runs it once with the one-launch device loop and once with
RS_ENGINE_LOOP=host (the per-kernel host loop, itself checked step for step against the
reference's engine.run in test_gpu_engine.py)."""
import hashlib
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

CASES = {
    # name: (n, generate_poisson rate, SchedulerConfig kwargs, DeviceEngine kwargs, run kwargs, cost preset)
    "calibrated": (5000, 40.0, dict(max_batch=64, starvation_threshold=30, priority_quantum=8),
                   dict(length_calibrated=True), {}, "default"),
    "non_preemptive": (5000, 40.0, dict(max_batch=48, starvation_threshold=20, priority_quantum=5, preemption=False),
                       {}, {}, "fast"),
    "stop_after": (5000, 40.0, dict(max_batch=128), {}, dict(stop_after_finished=1500), "default"),
    "time_limit": (5000, 40.0, dict(max_batch=128), {}, dict(time_limit_s=60.0), "default"),
    "max_batch_512": (8000, 200.0, dict(max_batch=512, starvation_threshold=50, priority_quantum=10), {}, {},
                      "default"),
    "no_predictor_charge": (4000, 80.0, dict(max_batch=256), dict(charges_predictor=False), {}, "unit"),
    "kv_budget": (3000, 40.0, dict(max_batch=64), dict(kv_budget=20000), {}, "default"),  # host loop either way
    # every request at t = 0: the first step admits 6000 rows (admission in 1024-row chunks)
    "burst": (6000, None, dict(max_batch=200, starvation_threshold=40, priority_quantum=6), {}, {}, "fast"),
    "max_batch_1": (600, 40.0, dict(max_batch=1, starvation_threshold=5, priority_quantum=2), {}, {}, "fast"),
}


def main(name):
    import numpy as np
    from paper_2408_15792_b200 import engine
    from paper_2408_15792_b200.schedulers import SchedulerConfig
    from paper_2408_15792_b200.workload import LengthDist, generate_burst, generate_poisson
    n, rate, sk, ek, rk, cost = CASES[name]
    if rate is None:
        reqs = list(generate_burst(n, LengthDist.parse("sharegpt"), seed=11, prompt_noise=0.25))
    else:
        reqs = list(generate_poisson(rate, n, LengthDist.parse("sharegpt"), seed=11, prompt_noise=0.25))
    scores = np.random.default_rng(12).normal(size=n)
    eng = engine.DeviceEngine(reqs, scores, SchedulerConfig(**sk), engine.COST_PRESETS[cost], **ek)
    res = eng.run(**rk)
    rows = hashlib.sha256(json.dumps(res.requests, sort_keys=True).encode()).hexdigest()
    print(json.dumps({"rows": rows, "metrics": res.metrics, "steps": res.steps}, sort_keys=True))


if __name__ == "__main__":
    main(sys.argv[1])

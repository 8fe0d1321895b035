"""Record reference engine runs (ranksched.engine.run, policy "ranking") as fixtures for
the device engine (paper_2408_15792_b200.engine). Run in the build container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_engine_golden.py

The scorer is a deterministic score table (a stand-in for the OPT ranker's cached
scores: fp32 values widened to float64, with ties), so the reference's decisions are
a function of the trace and the table only. Stored per case: the trace fields the
engine reads, the score table, the reference's metrics and per-request rows, and the
sha256 of its canonical step records (engine.py:96-101) plus the first records in full.
"""

from __future__ import annotations

import hashlib
import json
import pathlib
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
from ranksched import engine  # noqa: E402
from ranksched.predictors import Scorer  # noqa: E402
from ranksched.schedulers import SchedulerConfig  # noqa: E402
from ranksched.workload import LengthDist, generate_poisson  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parent / "engine_golden.json"


class TableScorer(Scorer):
    kind = "table"
    length_calibrated = False
    charges_predictor = True

    def __init__(self, table):
        self.table = table

    def score_batch(self, requests, seed):
        return [self.table[r.id] for r in requests]

    def to_dict(self):
        return {"kind": self.kind}


def canonical(obj) -> str:
    return json.dumps(obj, sort_keys=True, separators=(",", ":"))


def case(tag, n, rate, dist, seed, sched, cost, kv_budget=None, ties=False):
    trace = generate_poisson(rate, n, LengthDist.parse(dist), seed, prompt_noise=0.25)
    rng = np.random.default_rng(seed + 100)
    sc = rng.normal(size=n).astype(np.float32)
    if ties:
        sc = np.round(sc * 4) / 4
    table = {r.id: float(sc[k]) for k, r in enumerate(trace.requests)}
    res = engine.run(trace, "ranking", TableScorer(table), sched, engine.COST_PRESETS[cost], kv_budget=kv_budget)
    recs = res.records
    return {
        "tag": tag, "sched": {"max_batch": sched.max_batch, "starvation_threshold": sched.starvation_threshold,
                              "priority_quantum": sched.priority_quantum, "preemption": sched.preemption},
        "cost": cost, "kv_budget": kv_budget,
        "requests": [[r.id, r.arrival_time, r.prompt_tokens, r.true_output_tokens] for r in trace.requests],
        "scores": [table[r.id] for r in trace.requests],
        "metrics": res.metrics, "rows": res.requests, "n_steps": len(recs),
        "records_sha256": hashlib.sha256(canonical(recs).encode()).hexdigest(),
        "first_records": recs[:25],
    }


def main():
    cases = [
        case("poisson300_b16_fast", 300, 200.0, "uniform(1,200)", 1, SchedulerConfig(max_batch=16), "fast"),
        case("poisson500_b32_starve", 500, 400.0, "lognormal(4.0,0.8)", 2,
             SchedulerConfig(max_batch=32, starvation_threshold=20, priority_quantum=5), "fast", ties=True),
        case("poisson400_b24_kv", 400, 300.0, "uniform(1,300)", 5,
             SchedulerConfig(max_batch=24, starvation_threshold=10, priority_quantum=3), "fast", kv_budget=420),
        case("poisson200_nonpreempt", 200, 100.0, "uniform(1,100)", 4,
             SchedulerConfig(max_batch=8, starvation_threshold=15, priority_quantum=4, preemption=False), "default"),
    ]
    OUT.write_text(json.dumps({"generator": "make_engine_golden.py", "cases": cases}) + "\n")
    for c in cases:
        print(c["tag"], c["n_steps"], "steps", c["metrics"]["n_finished"], "finished",
              c["metrics"]["n_dropped"], "dropped", c["metrics"]["n_preemptions"], "preemptions")


def main_large():
    """The cfg5 shape at 20k requests (BASELINE configs[4] runs 100k: the reference loop
    takes ~6 min per 20k here): generate_poisson(40/s, sharegpt, seed 7, prompt_noise
    0.25), max_batch 256, starvation 100 / 50, the default cost preset. Stored compactly:
    the trace, the score table, the step count, sha256 of the canonical step records
    and of the per-request rows, and the metrics."""
    import time
    t0 = time.perf_counter()
    n, seed = 20000, 7
    trace = generate_poisson(40.0, n, LengthDist.parse("sharegpt"), seed, prompt_noise=0.25)
    rng = np.random.default_rng(seed + 100)
    sc = rng.normal(size=n).astype(np.float32)
    table = {r.id: float(sc[k]) for k, r in enumerate(trace.requests)}
    sched = SchedulerConfig(max_batch=256, starvation_threshold=100, priority_quantum=50)
    res = engine.run(trace, "ranking", TableScorer(table), sched, engine.COST_PRESETS["default"])
    recs = res.records
    out = {"generator": "make_engine_golden.py --large", "tag": "cfg5_poisson20k",
           "sched": {"max_batch": 256, "starvation_threshold": 100, "priority_quantum": 50, "preemption": True},
           "cost": "default", "kv_budget": None,
           "requests": [[r.id, r.arrival_time, r.prompt_tokens, r.true_output_tokens] for r in trace.requests],
           "scores": [table[r.id] for r in trace.requests], "metrics": res.metrics, "n_steps": len(recs),
           "records_sha256": hashlib.sha256(canonical(recs).encode()).hexdigest(),
           "rows_sha256": hashlib.sha256(canonical(res.requests).encode()).hexdigest(),
           "reference_seconds": time.perf_counter() - t0}
    (OUT.parent / "engine_golden_20k.json").write_text(json.dumps(out) + "\n")
    print(out["tag"], out["n_steps"], "steps", f"{out['reference_seconds']:.0f} s")


if __name__ == "__main__":
    main_large() if "--large" in sys.argv else main()

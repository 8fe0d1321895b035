"""Acceptance criterion 5 of the reference (test_acceptance.py:173-197: oracle-scored
ranking reproduces shortest-remaining-first decisions on 100 random traces) as a fixture:
the reference's own SRTF runs on the same 100 traces, decision fields only. The device
engine, given the true lengths as length-calibrated scores, must reproduce them. Run in
the build container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_srtf_golden.py
"""

from __future__ import annotations

import hashlib
import json
import pathlib
import random as pyrandom
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from ranksched.engine import COST_PRESETS, run  # noqa: E402
from ranksched.schedulers import SchedulerConfig  # noqa: E402
from ranksched.workload import LengthDist, generate_burst, generate_poisson  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parent / "srtf_golden.json"
FIELDS = ("now_ns", "iter_ns", "run", "preempted", "promoted", "demoted", "admitted", "dropped", "finished")


def main():
    rng = pyrandom.Random(55)
    dist = LengthDist.parse("uniform(1,40)")
    cases = []
    for i in range(100):
        n = rng.randint(3, 100)
        if i % 2:
            trace = generate_burst(n, dist, seed=1000 + i)
        else:
            trace = generate_poisson(rng.choice([2.0, 8.0]), n, dist, seed=1000 + i)
        mb = rng.choice([1, 2, 4, 8])
        kv = rng.choice([None, 200, 1000])
        res = run(trace, policy="srtf", sched=SchedulerConfig(max_batch=mb, starvation_threshold=0), kv_budget=kv,
                  cost=COST_PRESETS["fast"])
        dec = [{f: r[f] for f in FIELDS} for r in res.records]
        cases.append({"max_batch": mb, "kv_budget": kv,
                      "requests": [[r.id, r.arrival_time, r.prompt_tokens, r.true_output_tokens]
                                   for r in trace.requests],
                      "n_steps": len(dec),
                      "decisions_sha256": hashlib.sha256(json.dumps(dec, sort_keys=True,
                                                                    separators=(",", ":")).encode()).hexdigest(),
                      "metrics": res.metrics})
    OUT.write_text(json.dumps({"generator": "make_srtf_golden.py", "fields": FIELDS, "cases": cases}) + "\n")
    print(len(cases), "cases", sum(c["n_steps"] for c in cases), "steps")


if __name__ == "__main__":
    main()

"""Generate golden vectors by running the REFERENCE (ranksched 0.1.0) itself.

Run in the build container (where /root/reference exists):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py
Writes tests/golden/{tau,listmle,schedule}_golden.json. The fixtures are small and
committed; the GPU box never reads /root/reference. Large-n cases (1M rows) are
stored as a seeded recipe + the reference's outputs (see make_large_golden.py).
"""

from __future__ import annotations

import json
import math
import pathlib
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
from ranksched.ranking import kendall_tau_b, list_mle_gradient, list_mle_loss, bucket_lengths  # noqa: E402
from ranksched.schedulers import RankingPolicy, SchedulerConfig  # noqa: E402
from ranksched.workload import Request, RequestState  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parent


def tau_cases():
    cases = []

    def add(x, y, tag):
        r = kendall_tau_b(x, y)
        cases.append({"tag": tag, "x": [float(v) for v in x], "y": [float(v) for v in y], "tau": r.tau,
                      "concordant": r.concordant, "discordant": r.discordant, "n_pairs": r.n_pairs})

    # test_ranking.py:24-44 hand values and degenerate inputs
    add([1, 2, 3, 4], [1, 2, 4, 3], "hand_2/3")
    add([1, 2, 3], [1, 2, 3], "hand_+1")
    add([1, 2, 3], [3, 2, 1], "hand_-1")
    add([1, 1, 2], [1, 2, 2], "frozen_ties")
    add([10, 10, 20], [1, 2, 3], "spec_140")
    add([], [], "empty")
    add([1.0], [2.0], "single")
    add([1, 1, 1], [1, 2, 3], "x_all_tied")
    add([0.0, -0.0, 1.0], [1.0, 2.0, 3.0], "neg_zero_tie")
    # test_ranking.py:47-56 generator (rng 42, small alphabets -> ties)
    rng = np.random.default_rng(42)
    for _ in range(200):
        n = int(rng.integers(2, 40))
        add(rng.integers(0, 6, size=n), rng.integers(0, 6, size=n), "brute_ties")
    # test_acceptance.py:91-113 generator (rng 2024, three mixes)
    rng = np.random.default_rng(2024)
    for i in range(1000):
        n = int(rng.integers(2, 51))
        if i % 3 == 0:
            x = rng.integers(0, 8, n).astype(float)
            y = rng.integers(0, 8, n).astype(float)
        elif i % 3 == 1:
            x = rng.normal(size=n)
            y = rng.normal(size=n)
        else:
            x = rng.integers(0, 5, n).astype(float)
            y = rng.normal(size=n)
        add(x, y, "c02")
    for n in (2, 5, 17, 50):
        x = np.sort(rng.normal(size=n))
        add(x, np.exp(x), "c02_endpoint+1")
        add(x, -np.exp(x), "c02_endpoint-1")
    # medium sizes with heavy ties (lengths in [1, 2048], fp32 scores)
    rng = np.random.default_rng(5)
    for n in (1000, 4096, 10000):
        x = rng.normal(size=n).astype(np.float32)
        y = rng.integers(1, 2049, n)
        add(x.astype(np.float64), y.astype(np.float64), f"medium_{n}")
    return cases


def listmle_cases():
    cases = []

    def add(s, o, tag):
        s = np.asarray(s, dtype=np.float64)
        o = np.asarray(o, dtype=np.int64)
        cases.append({"tag": tag, "scores": s.tolist(), "order": o.tolist(),
                      "loss": list_mle_loss(s, o), "grad": list_mle_gradient(s, o).tolist()})

    add([0.0, 0.0], [0, 1], "hand_ln2")
    add([2.0, 1.0], [0, 1], "hand_margin")
    add([3.0], [0], "single")
    add([1000.0, 0.0], [0, 1], "large_0")
    add([0.0, 1000.0], [0, 1], "large_1000")
    add([1000.0, 0.0, -1000.0], [0, 1, 2], "large_grad")
    rng = np.random.default_rng(11)  # test_ranking.py:127-135
    for _ in range(100):
        n = int(rng.integers(1, 12))
        add(rng.normal(0, 3, size=n), rng.permutation(n), "brute")
    rng = np.random.default_rng(7)  # test_acceptance.py:119-134
    for _ in range(100):
        n = int(rng.integers(2, 33))
        add(rng.normal(0.0, 2.0, n), rng.permutation(n), "c03")
    rng = np.random.default_rng(8)
    for n in (64, 256, 1000):
        add(rng.normal(0.0, 3.0, n), rng.permutation(n), f"long_{n}")
    # training form (predictors.py:379-384): 64 lists x 32 (fp32 net outputs)
    rng = np.random.default_rng(9)
    g = rng.normal(0, 1, (64, 32)).astype(np.float32)
    lengths = rng.integers(1, 2049, (64, 32))
    losses, grads = [], []
    for k in range(64):
        order = np.argsort(bucket_lengths(lengths[k], 10), kind="stable")
        losses.append(list_mle_loss(g[k].astype(np.float64), order) / 32)
        grads.append((list_mle_gradient(g[k].astype(np.float64), order) / 32).tolist())
    train = {"g": g.tolist(), "lengths": lengths.tolist(), "width": 10, "loss": losses, "grad": grads}
    return cases, train


def _req(rid, arrival, prompt, gen, score, prio, starv, quantum, running):
    r = Request(id=rid, arrival_time=arrival, prompt_tokens=prompt, true_output_tokens=max(gen + 1, 10),
                prompt="", features=np.zeros(24))
    r.generated_tokens = gen
    r.score = score
    r.priority = prio
    r.starvation_count = starv
    r.quantum = quantum
    r.state = RequestState.RUNNING if running else RequestState.WAITING
    return r


def _state(reqs):
    return {"priority": [bool(r.priority) for r in reqs], "starvation": [r.starvation_count for r in reqs],
            "quantum": [r.quantum for r in reqs]}


def schedule_cases():
    cases = []
    rng = np.random.default_rng(123)
    for i in range(60):
        n = int(rng.integers(1, 300))
        ids = rng.permutation(10 * n)[:n].tolist()
        arrival = np.round(rng.uniform(0, 5, n), 1 if i % 2 else 3)
        score_mode = i % 4
        reqs = []
        for k in range(n):
            if score_mode == 0:
                s = float(rng.integers(0, 20))  # many ties
            elif score_mode == 1:
                s = float(rng.normal())
            elif score_mode == 2:
                s = float(np.float32(rng.normal()))
            else:
                s = float(rng.choice([0.0, -0.0, 1.5, -2.25]))
            if rng.random() < 0.1:
                s = None
            reqs.append(_req(ids[k], float(arrival[k]), int(rng.integers(1, 400)), int(rng.integers(0, 300)), s,
                             bool(rng.random() < 0.2), int(rng.integers(0, 6)), int(rng.integers(0, 4)),
                             bool(rng.random() < 0.4)))
        cfg = dict(max_batch=int(rng.choice([1, 2, 4, 8, 32, 256])), preemption=bool(i % 5 != 4),
                   starvation_threshold=int(rng.choice([0, 1, 3, 5, 100])),
                   priority_quantum=int(rng.choice([1, 2, 3, 50])))
        calibrated = bool(i % 3 == 0)
        kv = [None, 200, 1000, 5000][i % 4]
        pol = RankingPolicy(SchedulerConfig(**cfg), length_calibrated=calibrated)
        init = {"id": [r.id for r in reqs], "arrival": [r.arrival_time for r in reqs],
                "prompt": [r.prompt_tokens for r in reqs], "generated": [r.generated_tokens for r in reqs],
                "score": [r.score for r in reqs], "running": [r.state == RequestState.RUNNING for r in reqs],
                **_state(reqs)}
        steps = []
        for _ in range(4):
            d = pol.schedule(reqs, kv_budget=(1 << 62) if kv is None else kv)
            steps.append({"run": d.run, "promoted": d.promoted, "demoted": d.demoted, "state": _state(reqs)})
        cases.append({"config": cfg, "calibrated": calibrated, "kv_budget": kv, "init": init, "steps": steps})
    return cases


def main():
    (OUT / "tau_golden.json").write_text(json.dumps({"source": "ranksched.ranking.kendall_tau_b",
                                                     "cases": tau_cases()}))
    lm, train = listmle_cases()
    (OUT / "listmle_golden.json").write_text(json.dumps({"source": "ranksched.ranking.list_mle_*",
                                                         "cases": lm, "train": train}))
    (OUT / "schedule_golden.json").write_text(json.dumps({"source": "ranksched.schedulers.RankingPolicy",
                                                          "cases": schedule_cases()}))
    print("wrote", sorted(p.name for p in OUT.glob("*.json")))


if __name__ == "__main__":
    main()

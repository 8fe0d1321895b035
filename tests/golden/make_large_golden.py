"""Large-n golden vectors from the REFERENCE itself (build container only).

* tau at n = 1M (cfg4 recipe, fp32 and bf16-tie variants): the reference row loop
  (ranksched/ranking.py:45-50, verbatim numpy) partitioned by rows over P processes —
  C and D are sums over rows, so the partition does not change them — plus the
  reference's np.unique tie counts (ranking.py:52-57).
* one RankingPolicy.schedule step over the 1M queue recipe (unlimited KV and
  kv_budget = 10**6; ids in order and shuffled) with the reference's own classes.
Writes tests/golden/large_golden.json.
"""

from __future__ import annotations

import hashlib
import json
import multiprocessing as mp
import pathlib
import sys
import time

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent))
import recipes  # noqa: E402

REF = "/root/reference/pkg/src"
OUT = pathlib.Path(__file__).resolve().parent / "large_golden.json"


def _rows(args):
    variant, p, P = args
    x, y = recipes.tau_1m(variant)
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    n = len(x)
    c = d = 0
    for i in range(p, n - 1, P):  # ranking.py:45-50
        dx = np.sign(x[i + 1:] - x[i])
        dy = np.sign(y[i + 1:] - y[i])
        prod = dx * dy
        c += int(np.count_nonzero(prod > 0))
        d += int(np.count_nonzero(prod < 0))
    return c, d


def tau_golden(variant, P):
    t0 = time.time()
    with mp.Pool(P) as pool:
        parts = pool.map(_rows, [(variant, p, P) for p in range(P)])
    x, y = recipes.tau_1m(variant)

    def tied_pairs(v):  # ranking.py:52-54
        _, counts = np.unique(np.asarray(v, dtype=np.float64), return_counts=True)
        return int(np.sum(counts * (counts - 1) // 2))

    c = sum(p[0] for p in parts)
    d = sum(p[1] for p in parts)
    out = {"n": len(x), "concordant": c, "discordant": d, "n1": tied_pairs(x), "n2": tied_pairs(y),
           "seconds": time.time() - t0, "processes": P}
    print("tau", variant, out, flush=True)
    return out


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def schedule_golden(shuffled, kv):
    sys.path.insert(0, REF)
    from ranksched.schedulers import RankingPolicy, SchedulerConfig
    from ranksched.workload import Request, RequestState
    q = recipes.queue_1m(shuffled_ids=shuffled)
    n = len(q["ids"])
    feats = np.zeros(24)
    reqs = []
    for k in range(n):
        r = Request(id=int(q["ids"][k]), arrival_time=float(q["arrival"][k]), prompt_tokens=int(q["prompt"][k]),
                    true_output_tokens=1000, prompt="", features=feats)
        r.generated_tokens = int(q["generated"][k])
        r.score = float(q["score"][k])
        r.priority = bool(q["priority"][k])
        r.starvation_count = int(q["starvation"][k])
        r.quantum = int(q["quantum"][k])
        if q["running"][k]:
            r.state = RequestState.RUNNING
        reqs.append(r)
    pol = RankingPolicy(SchedulerConfig(max_batch=256, starvation_threshold=100, priority_quantum=50),
                        length_calibrated=False)
    t0 = time.time()
    d = pol.schedule(reqs, kv_budget=(1 << 62) if kv is None else kv)
    dt = time.time() - t0
    pr = np.array([r.priority for r in reqs], dtype=np.uint8)
    st = np.array([r.starvation_count for r in reqs], dtype=np.int32)
    qu = np.array([r.quantum for r in reqs], dtype=np.int32)
    out = {"shuffled_ids": shuffled, "kv_budget": kv, "run": d.run, "n_promoted": len(d.promoted),
           "n_demoted": len(d.demoted), "promoted_digest": _digest(np.array(d.promoted, dtype=np.int64)),
           "demoted_digest": _digest(np.array(d.demoted, dtype=np.int64)),
           "state_digest": _digest(pr, st, qu), "seconds": dt}
    print("schedule", shuffled, kv, {k: v for k, v in out.items() if k != "run"}, flush=True)
    return out


def main():
    P = int(sys.argv[1]) if len(sys.argv) > 1 else mp.cpu_count()
    what = sys.argv[2] if len(sys.argv) > 2 else "all"
    res = json.loads(OUT.read_text()) if OUT.exists() else {}
    if what in ("all", "schedule"):
        res["schedule"] = [schedule_golden(s, kv) for s in (False, True) for kv in (None, 60_000)]
    if what in ("all", "tau"):
        res["tau"] = {v: tau_golden(v, P) for v in ("f32", "bf16")}
    OUT.write_text(json.dumps(res))
    print("wrote", OUT)


if __name__ == "__main__":
    main()

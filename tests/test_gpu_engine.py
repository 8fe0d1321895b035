"""Device-resident engine loop (paper_2408_15792_b200.engine) vs the reference's own
engine.run(trace, "ranking", scorer) on the same traces and scores: step records
(run / preempted / promoted / demoted / admitted / dropped / finished / scored /
predictor_ns / iter_ns / now_ns) bit-identical (sha256 of the canonical records),
per-request rows and metrics equal. Fixtures: tests/golden/make_engine_golden.py."""

import hashlib
import json

import pytest

pytestmark = pytest.mark.gpu


def _canonical(obj):
    return json.dumps(obj, sort_keys=True, separators=(",", ":"))


@pytest.mark.parametrize("in_place", [False, True])
@pytest.mark.parametrize("idx", [0, 1, 2, 3])
def test_engine_matches_reference_run(golden, idx, in_place):
    from paper_2408_15792_b200 import engine
    from paper_2408_15792_b200.schedulers import SchedulerConfig
    from paper_2408_15792_b200.workload import Request
    c = golden["engine_golden"]["cases"][idx]
    reqs = [Request(id=i, arrival_time=a, prompt_tokens=p, true_output_tokens=o) for i, a, p, o in c["requests"]]
    sched = SchedulerConfig(**c["sched"])
    res = engine.run(reqs, scores=c["scores"], sched=sched, cost=engine.COST_PRESETS[c["cost"]],
                     kv_budget=c["kv_budget"], record=True, in_place_compaction=in_place)
    assert res.records[:len(c["first_records"])] == c["first_records"]
    assert len(res.records) == c["n_steps"]
    assert hashlib.sha256(_canonical(res.records).encode()).hexdigest() == c["records_sha256"]
    assert res.requests == c["rows"]
    for k, v in c["metrics"].items():
        assert res.metrics[k] == v, (k, res.metrics[k], v)


def test_engine_rejects_bad_config():
    from paper_2408_15792_b200 import engine
    from paper_2408_15792_b200.workload import Request
    reqs = [Request(id=0, arrival_time=0.0, prompt_tokens=1, true_output_tokens=1)]
    with pytest.raises(ValueError):
        engine.run(reqs, scores=[0.0], kv_budget=0)
    with pytest.raises(ValueError):
        engine.run(reqs)  # no scorer, no scores
    with pytest.raises(ValueError):
        engine.run(reqs, scores=[float("nan")])


def test_engine_out_of_place_matches_in_place_at_scale():
    """Thousands of alive rows (multi-CTA compaction, many preemptions): the out-of-place
    step gives the same records as the single-CTA in-place one."""
    import numpy as np
    from paper_2408_15792_b200 import engine
    from paper_2408_15792_b200.schedulers import SchedulerConfig
    from paper_2408_15792_b200.workload import Request
    rng = np.random.default_rng(3)
    n = 6000
    arr = np.cumsum(rng.exponential(1.0 / 200.0, n))
    out = np.clip(np.rint(rng.lognormal(5.0, 0.9, n)), 1, 2048).astype(int)
    reqs = [Request(id=i, arrival_time=float(arr[i]), prompt_tokens=int(rng.integers(8, 129)),
                    true_output_tokens=int(out[i])) for i in range(n)]
    scores = rng.normal(size=n).round(2).tolist()  # ties exercise the arrival tie-break
    sched = SchedulerConfig(max_batch=64, starvation_threshold=20, priority_quantum=5)
    a = engine.run(reqs, scores=scores, sched=sched, record=True, stop_after_finished=1500)
    b = engine.run(reqs, scores=scores, sched=sched, record=True, stop_after_finished=1500, in_place_compaction=True)
    assert max(len(r["preempted"]) for r in a.records) > 0
    assert a.steps == b.steps and a.records == b.records and a.requests == b.requests


def test_engine_mass_preemption_keeps_alive_order():
    """More preemptions in one step than the shared-memory ordering holds (4096): the
    ordered-scan path must still emit them in alive (= admission = id) order."""
    from paper_2408_15792_b200 import engine
    from paper_2408_15792_b200.schedulers import SchedulerConfig
    from paper_2408_15792_b200.workload import Request
    n1 = 6000
    reqs = [Request(id=i, arrival_time=0.0, prompt_tokens=4, true_output_tokens=50) for i in range(n1)]
    reqs += [Request(id=n1 + i, arrival_time=1e-3, prompt_tokens=4, true_output_tokens=50) for i in range(n1)]
    scores = [1.0] * n1 + [0.0] * n1  # the second burst outranks the first
    sched = SchedulerConfig(max_batch=n1, starvation_threshold=0, priority_quantum=50)
    for in_place in (False, True):
        res = engine.run(reqs, scores=scores, sched=sched, record=True, stop_after_finished=1,
                         in_place_compaction=in_place)
        pre = [r["preempted"] for r in res.records if r["preempted"]]
        assert pre and len(pre[0]) == n1 and pre[0] == sorted(pre[0]) == list(range(n1))


def test_engine_matches_reference_at_cfg5_scale():
    """20k Poisson(40/s) sharegpt requests with the cfg5 scheduler settings (BASELINE
    configs[4] at a fifth of its size): every step record and request row bit-identical
    to the reference engine's (fixture: make_engine_golden.py --large)."""
    import pathlib
    from paper_2408_15792_b200 import engine
    from paper_2408_15792_b200.schedulers import SchedulerConfig
    from paper_2408_15792_b200.workload import Request
    p = pathlib.Path(__file__).resolve().parent / "golden" / "engine_golden_20k.json"
    if not p.exists():
        pytest.skip("large engine golden not generated")
    c = json.loads(p.read_text())
    reqs = [Request(id=i, arrival_time=a, prompt_tokens=pt, true_output_tokens=o) for i, a, pt, o in c["requests"]]
    res = engine.run(reqs, scores=c["scores"], sched=SchedulerConfig(**c["sched"]),
                     cost=engine.COST_PRESETS[c["cost"]], record=True)
    assert len(res.records) == c["n_steps"]
    assert hashlib.sha256(_canonical(res.records).encode()).hexdigest() == c["records_sha256"]
    assert hashlib.sha256(_canonical(res.requests).encode()).hexdigest() == c["rows_sha256"]
    for k, v in c["metrics"].items():
        assert res.metrics[k] == v, (k, res.metrics[k], v)


class _OracleScores:
    """The reference's OracleScorer (predictors.py:53-60): score = true output length,
    length calibrated, no predictor charge."""

    kind = "oracle"
    length_calibrated = True
    charges_predictor = False

    def score_batch(self, requests, seed):
        return [float(r.true_output_tokens) for r in requests]


def test_oracle_ranking_reproduces_reference_srtf():
    """Acceptance criterion 5 (test_acceptance.py:173-197) across implementations: the
    device engine's ranking policy with oracle scores reproduces the reference's own
    SRTF decisions (now / iter / run / preempted / promoted / demoted / admitted /
    dropped / finished, every step) and metrics on its 100 random traces."""
    import pathlib
    from paper_2408_15792_b200 import engine
    from paper_2408_15792_b200.schedulers import SchedulerConfig
    from paper_2408_15792_b200.workload import Request
    g = json.loads((pathlib.Path(__file__).resolve().parent / "golden" / "srtf_golden.json").read_text())
    fields = g["fields"]
    for i, c in enumerate(g["cases"]):
        reqs = [Request(id=r, arrival_time=a, prompt_tokens=p, true_output_tokens=o) for r, a, p, o in c["requests"]]
        res = engine.run(reqs, scorer=_OracleScores(), sched=SchedulerConfig(max_batch=c["max_batch"],
                                                                            starvation_threshold=0),
                         kv_budget=c["kv_budget"], cost=engine.COST_PRESETS["fast"], record=True)
        dec = [{f: rec[f] for f in fields} for rec in res.records]
        assert len(dec) == c["n_steps"], i
        assert hashlib.sha256(_canonical(dec).encode()).hexdigest() == c["decisions_sha256"], i
        for k, v in c["metrics"].items():
            assert res.metrics[k] == v, (i, k, res.metrics[k], v)


@pytest.mark.parametrize("idx", [0, 1, 2, 3])
def test_engine_native_loop_matches_reference(golden, idx):
    """record=False runs the loop natively (rs_engine_run): same rows and metrics as the
    reference's engine.run on the recorded traces."""
    from paper_2408_15792_b200 import engine
    from paper_2408_15792_b200.schedulers import SchedulerConfig
    from paper_2408_15792_b200.workload import Request
    c = golden["engine_golden"]["cases"][idx]
    reqs = [Request(id=i, arrival_time=a, prompt_tokens=p, true_output_tokens=o) for i, a, p, o in c["requests"]]
    res = engine.run(reqs, scores=c["scores"], sched=SchedulerConfig(**c["sched"]),
                     cost=engine.COST_PRESETS[c["cost"]], kv_budget=c["kv_budget"])
    assert res.records == [] and res.steps == c["n_steps"]
    assert res.requests == c["rows"]
    for k, v in c["metrics"].items():
        assert res.metrics[k] == v, (k, res.metrics[k], v)


def test_engine_native_loop_at_cfg5_scale():
    import pathlib
    from paper_2408_15792_b200 import engine
    from paper_2408_15792_b200.schedulers import SchedulerConfig
    from paper_2408_15792_b200.workload import Request
    p = pathlib.Path(__file__).resolve().parent / "golden" / "engine_golden_20k.json"
    c = json.loads(p.read_text())
    reqs = [Request(id=i, arrival_time=a, prompt_tokens=pt, true_output_tokens=o) for i, a, pt, o in c["requests"]]
    res = engine.run(reqs, scores=c["scores"], sched=SchedulerConfig(**c["sched"]),
                     cost=engine.COST_PRESETS[c["cost"]])
    assert res.steps == c["n_steps"]
    assert hashlib.sha256(_canonical(res.requests).encode()).hexdigest() == c["rows_sha256"]
    for k, v in c["metrics"].items():
        assert res.metrics[k] == v, (k, res.metrics[k], v)


def test_engine_rescore_hook_matches_cache(golden):
    """The per-step re-score hook (re-scoring every alive request, reference rescore=True
    mode) gives the cached run's decisions when the scorer is a pure function."""
    import torch
    from paper_2408_15792_b200 import engine
    from paper_2408_15792_b200.schedulers import SchedulerConfig
    from paper_2408_15792_b200.workload import Request
    c = golden["engine_golden"]["cases"][1]
    reqs = [Request(id=i, arrival_time=a, prompt_tokens=p, true_output_tokens=o) for i, a, p, o in c["requests"]]
    table = torch.tensor(c["scores"], dtype=torch.float64, device="cuda")
    calls = []

    def rescore(alive):
        calls.append(alive.numel())
        return table[alive]

    kw = dict(sched=SchedulerConfig(**c["sched"]), cost=engine.COST_PRESETS[c["cost"]])
    a = engine.DeviceEngine(reqs, c["scores"], **kw).run(max_steps=60, record=True)
    b = engine.DeviceEngine(reqs, c["scores"], **kw).run(max_steps=60, record=True, rescore=rescore)
    assert len(calls) == a.steps == b.steps == 60 and sum(calls) > 0
    assert a.records == b.records and a.requests == b.requests

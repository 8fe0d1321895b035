"""K9 rank-step on the B200 vs the reference: run / promoted / demoted / state bit-exact."""

import hashlib

import numpy as np
import pytest
import torch

from test_oracle_golden import schedule_requests

pytestmark = pytest.mark.gpu


def test_schedule_golden_multi_step(golden):
    from paper_2408_15792_b200.schedulers import RankingPolicy, SchedulerConfig
    for ci, case in enumerate(golden["schedule_golden"]["cases"]):
        pol = RankingPolicy(SchedulerConfig(**case["config"]), length_calibrated=case["calibrated"])
        reqs = schedule_requests(case["init"])
        kv = (1 << 62) if case["kv_budget"] is None else case["kv_budget"]
        for si, step in enumerate(case["steps"]):
            d = pol.schedule(reqs, kv)
            assert (d.run, d.promoted, d.demoted) == (step["run"], step["promoted"], step["demoted"]), (ci, si)
            assert [bool(r.priority) for r in reqs] == step["state"]["priority"], (ci, si)
            assert [r.starvation_count for r in reqs] == step["state"]["starvation"], (ci, si)
            assert [r.quantum for r in reqs] == step["state"]["quantum"], (ci, si)


def _mk(rid, arrival=0.0, prompt=4, gen=0, score=None, prio=False, starv=0, quantum=0, running=False):
    from paper_2408_15792_b200.workload import Request, RequestState
    r = Request(id=rid, arrival_time=arrival, prompt_tokens=prompt, true_output_tokens=max(10, gen + 1))
    r.generated_tokens, r.score, r.priority, r.starvation_count, r.quantum = gen, score, prio, starv, quantum
    r.state = RequestState.RUNNING if running else RequestState.WAITING
    return r


def test_reference_unit_cases():
    """test_schedulers.py:211-321 restated against the device policy."""
    from paper_2408_15792_b200.schedulers import RankingPolicy, SchedulerConfig
    big = 10 ** 9
    pol = RankingPolicy(SchedulerConfig(starvation_threshold=0), True)
    assert pol.schedule([_mk(0, score=30.0), _mk(1, score=5.0), _mk(2, score=12.0)], big).run == [1, 2, 0]
    assert pol.schedule([_mk(0, 0.0, score=1.0), _mk(1, 2.0), _mk(2, 1.0)], big).run == [2, 1, 0]
    assert pol.schedule([_mk(0, score=1.0), _mk(1, score=99.0, prio=True, quantum=5)], big).run == [1, 0]
    assert pol.schedule([_mk(2, 1.0, score=7.0), _mk(1, 1.0, score=7.0), _mk(0, 2.0, score=7.0)], big).run == [1, 2, 0]
    cal = RankingPolicy(SchedulerConfig(starvation_threshold=0, max_batch=1), True)
    assert cal.schedule([_mk(0, score=50.0, gen=45, running=True), _mk(1, score=10.0)], big).run == [0]
    raw = RankingPolicy(SchedulerConfig(starvation_threshold=0, max_batch=1), False)
    assert raw.schedule([_mk(0, score=50.0, gen=45, running=True), _mk(1, score=10.0)], big).run == [1]
    # alternation trace d1..d4 (test_schedulers.py:271-287)
    pol = RankingPolicy(SchedulerConfig(max_batch=1, starvation_threshold=1, priority_quantum=1), True)
    a, b = _mk(0, score=10.0), _mk(1, score=10.0)
    want = [([0], [1], []), ([1], [0], [1]), ([0], [1], [0]), ([1], [0], [1])]
    for w in want:
        d = pol.schedule([a, b], big)
        assert (d.run, d.promoted, d.demoted) == tuple(map(list, w))
    # KV: skip oversized but keep going; need includes generated tokens
    pol = RankingPolicy(SchedulerConfig(max_batch=8, starvation_threshold=0), True)
    cands = [_mk(0, 0.0, prompt=100, score=1.0), _mk(1, 1.0, prompt=400, score=2.0), _mk(2, 2.0, prompt=50, score=3.0)]
    assert pol.schedule(cands, 200).run == [0, 2]
    r = _mk(0, prompt=10, gen=30, score=1.0)
    assert pol.schedule([r], 40).run == [] and pol.schedule([r], 41).run == [0]


def _queue_from_recipe(q, dev):
    from paper_2408_15792_b200.schedulers import DeviceQueue
    return DeviceQueue.from_arrays(score=q["score"], scored=np.ones(len(q["ids"]), bool), priority=q["priority"],
                                   running=q["running"], prompt_tokens=q["prompt"], generated_tokens=q["generated"],
                                   arrival_time=q["arrival"], ids=q["ids"], starvation=q["starvation"],
                                   quantum=q["quantum"], dev=dev)


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def test_schedule_1m_matches_reference(golden):
    import recipes
    from paper_2408_15792_b200.schedulers import SchedulerConfig
    if "large_golden" not in golden:
        pytest.skip("large golden not generated")
    cfg = SchedulerConfig(max_batch=256, starvation_threshold=100, priority_quantum=50)
    for g in golden["large_golden"]["schedule"]:
        q = recipes.queue_1m(shuffled_ids=g["shuffled_ids"])
        dq = _queue_from_recipe(q, torch.device("cuda"))
        dq.rank_step(cfg, g["kv_budget"], length_calibrated=False)
        d = dq.decision()
        assert d.run == g["run"]
        assert len(d.promoted) == g["n_promoted"] and len(d.demoted) == g["n_demoted"]
        assert _digest(np.array(d.promoted, dtype=np.int64)) == g["promoted_digest"]
        assert _digest(np.array(d.demoted, dtype=np.int64)) == g["demoted_digest"]
        pr = ((dq.flags.cpu().numpy() & 2) != 0).astype(np.uint8)
        assert _digest(pr, dq.starvation.cpu().numpy(), dq.quantum.cpu().numpy()) == g["state_digest"]


def test_schedule_random_vs_oracle_large():
    """Random 200k queues with heavy score ties, None scores and a KV budget."""
    from oracle import schedule_oracle as so
    from paper_2408_15792_b200.schedulers import RankingPolicy, SchedulerConfig
    rng = np.random.default_rng(99)
    n = 200_000
    for kv, calib in ((None, False), (3_000_000, True)):
        dev_reqs, ora_reqs = [], []
        scores = rng.integers(0, 50, n).astype(float)
        for k in range(n):
            kw = dict(rid=int(k * 7 % n), arrival=float(rng.integers(0, 1000)), prompt=int(rng.integers(1, 500)),
                      gen=int(rng.integers(0, 100)), score=None if rng.random() < 0.05 else float(scores[k]),
                      prio=bool(rng.random() < 0.02), starv=int(rng.integers(0, 100)), quantum=int(rng.integers(0, 3)),
                      running=bool(rng.random() < 0.3))
            dev_reqs.append(_mk(**kw))
            ora_reqs.append(_mk(**kw))
        cfg = SchedulerConfig(max_batch=1000, starvation_threshold=100, priority_quantum=50)
        d = RankingPolicy(cfg, calib).schedule(dev_reqs, (1 << 62) if kv is None else kv)
        run, prom, dem = so.schedule(ora_reqs, (1 << 62) if kv is None else kv, max_batch=1000, threshold=100,
                                     quantum=50, calibrated=calib)
        assert (d.run, d.promoted, d.demoted) == (run, prom, dem)
        assert [(r.priority, r.starvation_count, r.quantum) for r in dev_reqs] == \
            [(r.priority, r.starvation_count, r.quantum) for r in ora_reqs]


@pytest.mark.parametrize("n,max_batch,dist", [(3000, 256, "normal"), (5000, 256, "normal"), (100_000, 256, "ties"),
                                              (300_000, 256, "ties"), (1 << 20, 1024, "normal"),
                                              (50_000, 2048, "bf16"), (10_000, 1, "ties"),
                                              # >= 2^23 rows: level 0 keeps the candidates itself (one
                                              # column pass); "const" overflows the kept slices (fallback)
                                              ((1 << 23) + 5, 256, "normal"), (1 << 23, 1024, "ties"),
                                              (1 << 23, 256, "const"), ((1 << 23) + 3, 512, "bf16")])
def test_topk_select_matches_full_sort(n, max_batch, dist):
    """Unlimited KV uses the radix top-k select; a budget that never binds takes the
    full-sort path. Both must give the same batch, promotions and state."""
    import torch
    from paper_2408_15792_b200 import _lib
    from paper_2408_15792_b200.schedulers import DeviceQueue, SchedulerConfig
    rng = np.random.default_rng(n + max_batch)
    if dist == "normal":
        score = rng.normal(size=n).astype(np.float32).astype(np.float64)
    elif dist == "ties":
        score = rng.integers(0, 7, n).astype(np.float64)
    elif dist == "const":
        score = np.full(n, 0.5)
    else:
        score = rng.normal(size=n).astype(np.float32)
        score = (score.view(np.uint32) & 0xFFFF0000).view(np.float32).astype(np.float64)
    kw = dict(score=score, scored=rng.random(n) > 0.01, priority=rng.random(n) < 0.02, running=rng.random(n) < 0.3,
              prompt_tokens=rng.integers(1, 100, n).astype(np.int32),
              generated_tokens=rng.integers(0, 100, n).astype(np.int32), arrival_time=rng.random(n) * 100,
              ids=rng.permutation(n).astype(np.int64), starvation=rng.integers(0, 100, n).astype(np.int32),
              quantum=rng.integers(0, 3, n).astype(np.int32))
    cfg = SchedulerConfig(max_batch=max_batch, starvation_threshold=50, priority_quantum=5)
    out = []
    for kv in (None, 1 << 60):
        q = DeviceQueue.from_arrays(**kw)
        q.rank_step(cfg, kv, length_calibrated=False)
        d = q.decision()
        out.append((d, q.flags.cpu().numpy().copy(), q.starvation.cpu().numpy().copy(), q.quantum.cpu().numpy().copy()))
    (d0, f0, s0, q0), (d1, f1, s1, q1) = out
    assert d0.run == d1.run and len(d0.run) == min(n, max_batch)
    assert d0.promoted == d1.promoted and d0.demoted == d1.demoted
    assert (f0 == f1).all() and (s0 == s1).all() and (q0 == q1).all()


@pytest.mark.parametrize("n", [40_000, 200_000, 1 << 20])
def test_rank_step_graph_replay_equals_eager(n):
    """The CUDA-graph replay of a rank step (40k / 200k rows: the cooperative fused select;
    1M: the multi-launch select) equals two eager steps: batch, promotions and state."""
    import torch
    from paper_2408_15792_b200.schedulers import DeviceQueue, SchedulerConfig
    rng = np.random.default_rng(n)
    kw = dict(score=rng.normal(size=n), scored=rng.random(n) > 0.01, priority=rng.random(n) < 0.02,
              running=rng.random(n) < 0.3, prompt_tokens=rng.integers(1, 100, n).astype(np.int32),
              generated_tokens=rng.integers(0, 100, n).astype(np.int32), arrival_time=rng.random(n) * 100,
              ids=rng.permutation(n).astype(np.int64), starvation=rng.integers(0, 100, n).astype(np.int32),
              quantum=rng.integers(0, 3, n).astype(np.int32))
    cfg = SchedulerConfig(max_batch=256, starvation_threshold=50, priority_quantum=5)
    for calib in (False, True):
        a = DeviceQueue.from_arrays(**kw, score_dtype=torch.float32)
        b = DeviceQueue.from_arrays(**kw, score_dtype=torch.float32)
        a.rank_step(cfg, None, length_calibrated=calib)
        a.rank_step(cfg, None, length_calibrated=calib)
        replay = b.rank_step_graph(cfg, None, length_calibrated=calib)  # one eager step + capture
        replay()
        torch.cuda.synchronize()
        da, db = a.decision(), b.decision()
        assert da.run == db.run and da.promoted == db.promoted and da.demoted == db.demoted
        for x, y in ((a.flags, b.flags), (a.starvation, b.starvation), (a.quantum, b.quantum)):
            assert torch.equal(x, y)

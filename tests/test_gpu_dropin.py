"""A17 on hardware: the reference's own engine.run (engine.py:382-460, the scoring block
:414-428 and the schedule call :430) drives the B200 scorer and ranking policy after
install(), unchanged.

The check: with install() active, ranksched.engine.run(trace, "ranking", OptRankerScorer)
— the device ranker scoring real Request prompts, the device RankingPolicy scheduling
every step, the device kendall_tau_b in the metrics — produces exactly the step records,
per-request rows and metrics of the reference's own stock run (no install, the reference
RankingPolicy and tau) fed the same scores. The scorer dict hashes into the run config
without a prior save_scorer()."""

import pytest

pytestmark = pytest.mark.gpu


def _fixed_scorer(scores):
    class Fixed:
        kind = "fixed"
        length_calibrated = False
        warmup_tokens = 0
        charges_predictor = True

        def score_batch(self, requests, seed):
            return [scores[r.id] for r in requests]

        def to_dict(self):
            return {"kind": self.kind}

    return Fixed()


@pytest.mark.parametrize("preemption,kv_budget", [(True, None), (False, 6000)])
def test_reference_engine_run_drives_device_path(ranksched, preemption, kv_budget):
    import paper_2408_15792_b200 as b200
    from paper_2408_15792_b200 import schedulers as b_sched
    from paper_2408_15792_b200.predictors import OptRankerScorer
    from paper_2408_15792_b200.ranker import OptRanker, RankerConfig
    wl = ranksched.workload
    trace = wl.generate_poisson(40.0, 400, wl.LengthDist.parse("sharegpt"), seed=7, prompt_noise=0.25)
    scorer = OptRankerScorer(OptRanker(RankerConfig.opt_125m(n_layers=2), seed=0), seq_len=128)
    scores = dict(zip([r.id for r in trace], scorer.score_batch(list(trace), 0)))
    sched = ranksched.schedulers.SchedulerConfig(max_batch=16, starvation_threshold=20, priority_quantum=5,
                                                 preemption=preemption)
    calls = {"schedule": 0}
    orig = b_sched.RankingPolicy.schedule

    def counting(self, candidates, kv):
        calls["schedule"] += 1
        return orig(self, candidates, kv)

    b200.install(ranksched)
    b_sched.RankingPolicy.schedule = counting
    try:
        res = ranksched.engine.run(trace, "ranking", scorer, sched=sched, kv_budget=kv_budget)
    finally:
        b_sched.RankingPolicy.schedule = orig
        b200.uninstall(ranksched)
    assert calls["schedule"] == len(res.records) > 100
    ref = ranksched.engine.run(trace, "ranking", _fixed_scorer(scores), sched=sched, kv_budget=kv_budget)
    assert res.records == ref.records
    assert res.requests == ref.requests
    assert res.metrics == ref.metrics
    assert res.config["scorer_hash"] and res.config["scorer_hash"] != ref.config["scorer_hash"]
    assert sum(len(r["promoted"]) for r in res.records) > 0  # the starvation bump was exercised


def test_rebound_functions_return_reference_classes(ranksched):
    import numpy as np
    import paper_2408_15792_b200 as b200
    b200.install(ranksched)
    try:
        r = ranksched.ranking.kendall_tau_b([1, 2, 3, 4], [1, 2, 4, 3])
        assert type(r) is ranksched.ranking.TauResult and (r.concordant, r.discordant) == (5, 1)
        pol = ranksched.engine.make_policy("ranking", ranksched.schedulers.SchedulerConfig(max_batch=2), False)
        reqs = [ranksched.workload.Request(id=k, arrival_time=float(k), prompt_tokens=4, true_output_tokens=3)
                for k in range(5)]
        for k, q in enumerate(reqs):
            q.score = float(-k)
        d = pol.schedule(reqs, 1 << 62)
        assert type(d) is ranksched.schedulers.BatchDecision and d.run == [4, 3]
        assert [q.starvation_count for q in reqs] == [1, 1, 1, 0, 0]
        loss = ranksched.predictors.list_mle_loss(np.array([1.0, 0.0]), np.array([0, 1]))
        assert abs(loss - np.log1p(np.exp(-1.0))) < 1e-15  # test_ranking.py:103-110
    finally:
        b200.uninstall(ranksched)

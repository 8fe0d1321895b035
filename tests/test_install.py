"""install() rebinds the reference's hot-path names (CPU: no kernel is called)."""

import pytest


def test_install_rebinds_reference_names(ranksched):
    import paper_2408_15792_b200 as b200
    from paper_2408_15792_b200 import ranking as b_rank, schedulers as b_sched
    orig_tau = ranksched.ranking.kendall_tau_b
    orig_mp = ranksched.engine.make_policy
    orig_load = ranksched.predictors.load_scorer
    b200.install(ranksched)
    try:
        tau = ranksched.ranking.kendall_tau_b
        assert tau is not orig_tau
        assert ranksched.engine.kendall_tau_b is tau and ranksched.kendall_tau_b is tau
        assert ranksched.predictors.list_mle_loss is b_rank.list_mle_loss
        assert ranksched.predictors.list_mle_gradient is b_rank.list_mle_gradient
        cfg = ranksched.schedulers.SchedulerConfig()
        pol = ranksched.engine.make_policy("ranking", cfg, False)
        assert isinstance(pol, b_sched.RankingPolicy)
        # results come back in the reference's own classes
        assert pol.decision_cls is ranksched.schedulers.BatchDecision
        # non-hot-path policies still come from the reference
        assert type(ranksched.engine.make_policy("fcfs", cfg)).__module__ == "ranksched.schedulers"
        with pytest.raises(ValueError):
            ranksched.predictors.scorer_from_dict({"kind": "nope"})
        assert ranksched.predictors.scorer_from_dict({"kind": "oracle"}).kind == "oracle"
        assert ranksched.predictors.load_scorer is not orig_load
    finally:
        b200.uninstall(ranksched)
    assert ranksched.ranking.kendall_tau_b is orig_tau
    assert ranksched.engine.make_policy is orig_mp
    assert ranksched.predictors.load_scorer is orig_load

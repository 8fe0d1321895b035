"""install() rebinds the reference's hot-path names (CPU: no kernel is called)."""

import sys

import pytest

REF = "/root/reference/pkg/src"


def test_install_rebinds_reference_names():
    import os
    if not os.path.isdir(REF):
        pytest.skip("reference not present (GPU box)")
    sys.path.insert(0, REF)
    try:
        import ranksched
        import ranksched.engine
        import ranksched.predictors
        import ranksched.ranking
        import paper_2408_15792_b200 as b200
        from paper_2408_15792_b200 import ranking as b_rank, schedulers as b_sched
        orig_tau = ranksched.ranking.kendall_tau_b
        orig_mp = ranksched.engine.make_policy
        b200.install(ranksched)
        try:
            assert ranksched.ranking.kendall_tau_b is b_rank.kendall_tau_b
            assert ranksched.engine.kendall_tau_b is b_rank.kendall_tau_b
            assert ranksched.predictors.list_mle_loss is b_rank.list_mle_loss
            assert ranksched.kendall_tau_b is b_rank.kendall_tau_b
            cfg = ranksched.schedulers.SchedulerConfig()
            assert isinstance(ranksched.engine.make_policy("ranking", cfg, False), b_sched.RankingPolicy)
            # non-hot-path policies still come from the reference
            assert type(ranksched.engine.make_policy("fcfs", cfg)).__module__ == "ranksched.schedulers"
            with pytest.raises(ValueError):
                ranksched.predictors.scorer_from_dict({"kind": "nope"})
            assert ranksched.predictors.scorer_from_dict({"kind": "oracle"}).kind == "oracle"
        finally:
            b200.uninstall(ranksched)
        assert ranksched.ranking.kendall_tau_b is orig_tau
        assert ranksched.engine.make_policy is orig_mp
    finally:
        sys.path.remove(REF)

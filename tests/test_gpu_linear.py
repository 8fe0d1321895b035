"""A2/A3 parity bridge: the reference's own 24-feature linear / MLP ranker on the device
(linear_ranker.py) against the staged reference (predictors.py:159-406).

* training: train_ranking_features reproduces the reference's train_ranking trajectory
  on the cfg1 (desk_burst) recipe — same split, shuffles, lists, init — so the learned
  parameters, every checkpoint's train loss and eval tau, and the report agree within
  float64 summation-order noise (BLAS dot products vs the kernel's loops);
* scoring: a reference-trained scorer loaded through to_dict / from_dict scores the cfg1
  prompts within rel 1e-12 of the reference, in the same order.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _desk_burst(ranksched):
    wl = ranksched.workload
    return wl.generate_burst(2000, wl.LengthDist.parse("lognormal(5.0,0.8)"), seed=11, prompt_noise=0.25)


@pytest.mark.parametrize("hidden", [0, 32])
def test_train_matches_reference(ranksched, hidden):
    from paper_2408_15792_b200.linear_ranker import FeatureTrainConfig, train_ranking_features
    trace = _desk_burst(ranksched)
    ref = ranksched.predictors.train_ranking(trace, ranksched.predictors.TrainConfig(seed=0, hidden=hidden))
    ours = train_ranking_features(trace, FeatureTrainConfig(seed=0, hidden=hidden))
    rr, ro = ref.report, ours.report
    assert (ro["kind"], ro["steps"], ro["n_train"], ro["n_eval"]) == (rr["kind"], rr["steps"], rr["n_train"],
                                                                        rr["n_eval"])
    assert len(ro["checkpoints"]) == len(rr["checkpoints"]) > 5
    for a, b in zip(ro["checkpoints"], rr["checkpoints"]):
        assert a["step"] == b["step"]
        assert abs(a["train_loss"] - b["train_loss"]) <= 1e-9 * max(1.0, abs(b["train_loss"]))
        assert abs(a["eval_tau"] - b["eval_tau"]) <= 1e-3
    assert abs(ro["eval_tau"] - rr["eval_tau"]) <= 1e-3
    # the output bias b gets the gradient sum(dg) = 0 up to rounding (ListMLE is shift
    # invariant), so it is float64 noise of order 1e-9 in both runs: absolute bar
    for p, q in zip(ours.scorer.params, ref.scorer.net.params):
        np.testing.assert_allclose(p, q, rtol=1e-7, atol=1e-7)
    np.testing.assert_allclose(ours.scorer.mean.cpu().numpy(), ref.scorer.standardizer.mean, rtol=1e-13)
    np.testing.assert_allclose(ours.scorer.std.cpu().numpy(), ref.scorer.standardizer.std, rtol=1e-13)
    d = ours.scorer.to_dict()
    assert set(d) == set(ref.scorer.to_dict())


def test_scores_match_reference_cfg1(ranksched, golden):
    """BASELINE configs[0]: the reference's default ranker on 64 prompts x 128 tokens."""
    from paper_2408_15792_b200.linear_ranker import RankingModelScorer
    wl = ranksched.workload
    ref = ranksched.predictors.train_ranking(_desk_burst(ranksched), ranksched.predictors.TrainConfig(seed=0)).scorer
    ours = RankingModelScorer.from_dict(ref.to_dict())
    rng = np.random.default_rng(0)
    n, toks = 64, 128
    prompts = [" ".join(wl._VOCAB[i] for i in rng.integers(0, len(wl._VOCAB), toks)) for _ in range(n)]
    lengths = rng.integers(1, 2049, n)
    reqs = [wl.Request(id=k, arrival_time=float(k), prompt_tokens=toks, true_output_tokens=int(lengths[k]),
                       prompt=prompts[k]) for k in range(n)]
    want = np.array(ref.score_batch(reqs, 0))
    got = np.array(ours.score_batch(reqs, 0))
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(got, golden["cfg1_golden"]["scores"], rtol=1e-12, atol=1e-12)
    assert np.array_equal(np.argsort(got, kind="stable"), np.argsort(want, kind="stable"))
    assert ours.to_dict()["params"] == ref.to_dict()["params"]


def test_bad_arguments():
    from paper_2408_15792_b200.linear_ranker import RankingModelScorer
    with pytest.raises(ValueError):
        RankingModelScorer([np.zeros(5), np.zeros(1)], 0, np.zeros(24), np.ones(24))

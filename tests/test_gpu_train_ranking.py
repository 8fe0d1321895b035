"""train_ranking (A10, predictors.py:347-406) on the B200: the reference's trainer
contract with the OPT-shape ranker (test_predictors.py:140-197 are the model: a
learnable trace is learned, scores are oriented shortest-first, loss falls while tau
rises, training is bitwise deterministic, an explicit eval trace is honoured, tiny
traces are rejected)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

WORDS = [f"w{k}" for k in range(12)]


def _trace(n, seed):
    """Requests whose output length is set by the prompt's first word (plus noise
    words), so the ranker can learn it from the token ids."""
    from paper_2408_15792_b200.workload import Request
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        k = int(rng.integers(0, len(WORDS)))
        filler = " ".join(f"x{int(v)}" for v in rng.integers(0, 500, int(rng.integers(2, 12))))
        prompt = f"{WORDS[k]} {filler}"
        out.append(Request(id=i, arrival_time=float(i), prompt_tokens=len(prompt.split()),
                           true_output_tokens=int(10 + 150 * k + rng.integers(0, 20)), prompt=prompt))
    return out


def _cfg(**kw):
    from paper_2408_15792_b200.predictors import TrainConfig
    from paper_2408_15792_b200.ranker import RankerConfig
    rc = RankerConfig.opt_125m(vocab=2048, max_pos=64, d_model=256, n_layers=2, n_heads=4, d_ffn=1024)
    base = dict(epochs=4, batch_size=32, learning_rate=2e-3, seq_len=32, checkpoint_every=10, ranker=rc, seed=0)
    base.update(kw)
    return TrainConfig(**base)


def test_train_ranking_learns_and_orients():
    from paper_2408_15792_b200.predictors import train_ranking
    from paper_2408_15792_b200.ranking import kendall_tau_b
    t = _trace(600, seed=7)
    res = train_ranking(t, _cfg())
    rep = res.report
    assert rep["n_train"] + rep["n_eval"] == 600
    assert rep["steps"] == 4 * len([s for s in range(0, 480, 32) if 480 - s >= 2])
    cps = rep["checkpoints"]
    assert len(cps) >= 5
    assert cps[-1]["train_loss"] < cps[0]["train_loss"]
    assert cps[-1]["eval_tau"] > cps[0]["eval_tau"]
    assert rep["eval_tau"] > 0.6, rep
    fresh = _trace(200, seed=8)
    scores = res.scorer.score_batch(fresh, seed=0)
    assert kendall_tau_b(scores, [r.true_output_tokens for r in fresh]).tau > 0.6
    # orientation: ascending score = predicted shortest first (test_predictors.py:151-158)
    reqs = sorted(fresh, key=lambda r: r.true_output_tokens)
    s = res.scorer.score_batch([reqs[0], reqs[-1]], seed=0)
    assert s[0] < s[1]


def test_train_ranking_deterministic_and_lists_per_step():
    from paper_2408_15792_b200.predictors import train_ranking
    t = _trace(300, seed=11)
    a = train_ranking(t, _cfg(epochs=2, seed=3))
    b = train_ranking(t, _cfg(epochs=2, seed=3))
    assert torch.equal(a.scorer.model.flat, b.scorer.model.flat)
    assert a.report == b.report
    c = train_ranking(t, _cfg(epochs=2, seed=3, lists_per_step=4))
    assert c.report["steps"] == -(-a.report["steps"] // 4)


def test_train_ranking_eval_trace_and_errors():
    from paper_2408_15792_b200.predictors import train_ranking
    res = train_ranking(_trace(100, seed=13), _cfg(epochs=1), eval_trace=_trace(40, seed=14))
    assert res.report["n_train"] == 100 and res.report["n_eval"] == 40
    with pytest.raises(ValueError):
        train_ranking(_trace(3, seed=1), _cfg())

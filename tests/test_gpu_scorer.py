"""OptRankerScorer honours the reference Scorer contract (predictors.py:35-51, 228-259)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_scorer_contract_and_round_trip(tmp_path):
    from oracle import opt_ranker
    from paper_2408_15792_b200.predictors import OptRankerScorer, load_scorer, save_scorer
    from paper_2408_15792_b200.ranker import OptRanker, RankerConfig
    from paper_2408_15792_b200.workload import Request, prompt_token_ids
    cfg = RankerConfig.opt_125m(n_layers=2)
    s = OptRankerScorer(OptRanker(cfg, seed=4), seq_len=64)
    assert (s.kind, s.length_calibrated, s.charges_predictor, s.warmup_tokens) == ("opt-ranker", False, True, 0)
    words = "list explain write code summarize why how the a of".split()
    rng = np.random.default_rng(0)
    reqs = [Request(id=k, arrival_time=0.0, prompt_tokens=5, true_output_tokens=10,
                    prompt=" ".join(rng.choice(words, size=int(rng.integers(1, 80)))))
            for k in range(37)]
    scores = s.score_batch(reqs, seed=0)
    assert len(scores) == 37 and all(isinstance(v, float) for v in scores)
    # orientation: score = -g, g from the oracle on the same ids / last positions
    enc = [prompt_token_ids(r.prompt, 64) for r in reqs]
    ids = np.stack([e[0] for e in enc])
    last = np.array([e[1] for e in enc])
    g_ref = opt_ranker.forward(s.model.params_cpu_fp32(), cfg, ids, last).numpy()
    np.testing.assert_allclose(-np.array(scores), g_ref, atol=1e-2 * max(1.0, np.abs(g_ref).max()))
    # deterministic and batch-independent
    assert s.score_batch(reqs, seed=5) == scores
    assert s.score_batch(reqs[3:4], seed=0) == scores[3:4]
    path = tmp_path / "scorer.json"
    save_scorer(s, str(path))
    s2 = load_scorer(str(path))
    assert s2.kind == "opt-ranker" and s2.score_batch(reqs, 0) == scores
    assert torch.equal(s2.model.flat, s.model.flat)

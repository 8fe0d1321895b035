"""rs_tokenize (prompt strings -> OPT ids on the device) vs the host map
workload.prompt_token_ids: identical ids and last positions, edge cases included."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

WS = [" ", "\t", "\n", "\r", "\x0b", "\x0c", "\x1c", "\x1d", "\x1e", "\x1f"]


def _host(prompts, S, vocab):
    from paper_2408_15792_b200.workload import prompt_token_ids
    out = [prompt_token_ids(p, S, vocab) for p in prompts]
    return np.stack([o[0] for o in out]), np.array([o[1] for o in out], dtype=np.int32)


def _random_prompts(rng, n, max_words):
    words = ["What", "is", "THE", "best", "way", "to", "write", "Python?", "x", "a-b", "9", "Long" * 20, "q!"]
    out = []
    for _ in range(n):
        k = int(rng.integers(0, max_words + 1))
        parts = []
        for _ in range(k):
            parts.append(words[int(rng.integers(len(words)))])
            parts.append("".join(WS[int(j)] for j in rng.integers(0, len(WS), int(rng.integers(1, 3)))))
        lead = WS[int(rng.integers(len(WS)))] if rng.random() < 0.3 else ""
        out.append(lead + "".join(parts))
    return out


@pytest.mark.parametrize("S,max_words", [(128, 40), (16, 200), (1, 5), (2048, 2600)])
def test_tokenize_matches_host_map(S, max_words):
    from paper_2408_15792_b200.workload import prompt_token_ids_device
    rng = np.random.default_rng(S + max_words)
    prompts = _random_prompts(rng, 300, max_words) + ["", "   ", "\t\n", "A", "  lead trail  ", "x " * 3000]
    ids, last = prompt_token_ids_device(prompts, S, 50272)
    want_ids, want_last = _host(prompts, S, 50272)
    np.testing.assert_array_equal(ids.cpu().numpy(), want_ids)
    np.testing.assert_array_equal(last.cpu().numpy(), want_last)


def test_tokenize_rejects_unicode_dependent_prompts():
    from paper_2408_15792_b200.workload import prompt_token_ids_device
    with pytest.raises(ValueError):
        prompt_token_ids_device(["plain", "cafÉ au lait"], 8)
    with pytest.raises(ValueError):
        prompt_token_ids_device(["no break"], 8)  # NBSP: Unicode whitespace
    # non-ASCII past the kept tokens does not change the ids
    ids, _ = prompt_token_ids_device(["a b é"], 2)
    from paper_2408_15792_b200.workload import prompt_token_ids
    np.testing.assert_array_equal(ids.cpu().numpy()[0], prompt_token_ids("a b é", 2)[0])


def test_scorer_device_tokenizer_same_scores():
    from paper_2408_15792_b200.predictors import OptRankerScorer
    from paper_2408_15792_b200.ranker import RankerConfig
    from paper_2408_15792_b200.workload import Request
    rng = np.random.default_rng(1)
    cfg = RankerConfig(n_layers=1)
    reqs = [Request(id=i, arrival_time=float(i), prompt_tokens=5, true_output_tokens=5, prompt=p)
            for i, p in enumerate(_random_prompts(rng, 64, 30))]
    a = OptRankerScorer(cfg=cfg, seq_len=32, seed=0, device_tokenizer=False)
    b = OptRankerScorer(model=a.model, seq_len=32, device_tokenizer=True)
    assert a.score_batch(reqs, 0) == b.score_batch(reqs, 0)


def test_scorer_auto_tokenizer_patches_unicode_rows():
    """device_tokenizer='auto' (the default): ASCII prompts on the device, prompts needing
    Unicode-aware splitting through the host map, same ids / scores as the host map."""
    from paper_2408_15792_b200.predictors import OptRankerScorer
    from paper_2408_15792_b200.ranker import RankerConfig
    from paper_2408_15792_b200.workload import Request, prompt_token_ids, prompt_token_ids_device
    prompts = ["plain words here", "cafÉ au lait", "no\u00a0break space", "", "  x  ", "ÅNGSTRÖM units"]
    ids, last = prompt_token_ids_device(prompts, 8, host_fallback=True)
    for k, p in enumerate(prompts):
        want_ids, want_last = prompt_token_ids(p, 8)
        np.testing.assert_array_equal(ids[k].cpu().numpy(), want_ids)
        assert int(last[k]) == want_last
    reqs = [Request(id=i, arrival_time=0.0, prompt_tokens=3, true_output_tokens=3, prompt=p)
            for i, p in enumerate(prompts)]
    a = OptRankerScorer(cfg=RankerConfig(n_layers=1), seq_len=8, seed=0, device_tokenizer=False)
    b = OptRankerScorer(model=a.model, seq_len=8)
    assert b.device_tokenizer == "auto" and a.score_batch(reqs, 0) == b.score_batch(reqs, 0)

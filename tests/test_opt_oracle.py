"""oracle/opt_ranker.py (fp32) is pinned to transformers' OPTModel (CPU)."""

import numpy as np
import pytest
import torch

from oracle import opt_ranker
from opt_hf import hf_scores


def _cfg(**kw):
    # RankerConfig without loading the CUDA library (pure dataclass)
    from paper_2408_15792_b200.ranker import RankerConfig
    return RankerConfig.opt_125m(**kw)


@pytest.mark.parametrize("kw", [dict(vocab=1000, max_pos=128, d_model=256, n_layers=2, n_heads=4, d_ffn=1024),
                                dict(vocab=500, max_pos=64, d_model=128, n_layers=3, n_heads=2, d_ffn=256,
                                     activation=1)])
def test_opt_oracle_matches_transformers(kw):
    from paper_2408_15792_b200.ranker import init_params
    cfg = _cfg(**kw)
    params = init_params(cfg, seed=1)
    # make LayerNorm / bias paths non-trivial
    g = torch.Generator().manual_seed(2)
    for k in params:
        if k.endswith("_b") or "ln" in k:
            params[k] = params[k] + 0.1 * torch.randn(params[k].shape, generator=g)
    ids = torch.randint(0, cfg.vocab, (3, 40), generator=g)
    last = torch.tensor([39, 10, 0])
    got = opt_ranker.forward(params, cfg, ids.numpy(), last.numpy())
    want = hf_scores(cfg, params, ids, last)
    torch.testing.assert_close(got, want, rtol=1e-4, atol=1e-4)


def test_opt_125m_param_count():
    cfg = _cfg()
    # 125,239,296 OPTModel params + 769 head params
    assert cfg.n_params() == 125_240_065
    assert cfg.flops_per_prompt(512) == pytest.approx(9.1814e10, rel=1e-4)

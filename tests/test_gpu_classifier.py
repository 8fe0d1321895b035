"""§8f #4: the bucketed-classification baseline on the OPT backbone (reference:
ClassifierScorer / train_classifier, predictors.py:262-300, :409-479) — the head and
cross-entropy kernels vs torch fp32, rs_ranker_grad_cls vs torch autograd (same bar as
the ListMLE pass, tests/test_gpu_train.py), and train_classifier on a learnable trace."""

import numpy as np
import pytest
import torch

from test_gpu_train import _forward_with_grad, _small_cfg
from test_gpu_train_ranking import _cfg, _trace

pytestmark = pytest.mark.gpu


def test_head_and_cross_entropy_kernels():
    from paper_2408_15792_b200 import _lib
    _lib.device()
    g = torch.Generator(device="cuda").manual_seed(0)
    B, d, C = 37, 256, 7
    feat = torch.randn(B, d, device="cuda", generator=g)
    W = torch.randn(C, d, device="cuda", generator=g) * 0.1
    b = torch.randn(C, device="cuda", generator=g)
    lab = torch.randint(0, C, (B,), device="cuda", generator=g, dtype=torch.int32)
    lib, st = _lib.load(), _lib.stream_handle()
    logits = torch.empty(B, C, device="cuda")
    _lib.check(lib.rs_cls_logits(feat.data_ptr(), W.data_ptr(), b.data_ptr(), B, d, C, logits.data_ptr(), st))
    torch.testing.assert_close(logits, feat @ W.t() + b, rtol=1e-5, atol=1e-4)
    loss = torch.empty(B, device="cuda")
    dl = torch.empty(B, C, device="cuda")
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.check(lib.rs_cls_ce(logits.data_ptr(), lab.data_ptr(), B, C, loss.data_ptr(), dl.data_ptr(), bad.data_ptr(),
                             st))
    ref = torch.nn.functional.cross_entropy(logits, lab.long(), reduction="none")
    torch.testing.assert_close(loss, ref, rtol=1e-5, atol=1e-5)
    want = torch.softmax(logits, 1) - torch.nn.functional.one_hot(lab.long(), C).float()
    torch.testing.assert_close(dl, want, rtol=1e-5, atol=1e-6)
    assert bad.item() == 0
    lab[3] = C  # out of range
    _lib.check(lib.rs_cls_ce(logits.data_ptr(), lab.data_ptr(), B, C, loss.data_ptr(), dl.data_ptr(), bad.data_ptr(),
                             st))
    assert bad.item() == 1


@pytest.mark.parametrize("S,n,mb", [(64, 48, 16), (100, 40, 20)])
def test_classifier_gradient_matches_autograd(S, n, mb):
    from paper_2408_15792_b200.ranker import OptRanker, init_params
    from paper_2408_15792_b200.trainer import ClassifierTrainer
    cfg = _small_cfg()
    params = init_params(cfg, seed=5)
    g = torch.Generator().manual_seed(7)
    for k in params:
        if k.endswith("_b") or "ln" in k:
            params[k] = params[k] + 0.05 * torch.randn(params[k].shape, generator=g)
    model = OptRanker(cfg, params=params)
    C = 5
    tr = ClassifierTrainer(model, C, prompts_per_micro=mb)
    tr.head.copy_(0.05 * torch.randn(tr.head.shape, generator=g).cuda())
    ids = torch.randint(4, cfg.vocab, (n, S), generator=g, dtype=torch.int32)
    lab = torch.randint(0, C, (n,), generator=g, dtype=torch.int32)
    loss = tr.accumulate(ids.cuda(), lab.cuda()).cpu()
    # features of the inference path match the training pass's reference
    Wc, bc = tr.W.detach().clone(), tr.b.detach().clone()

    def ref(emulate):
        rp = {k: v.cuda().clone().requires_grad_(True) for k, v in model.params_cpu_fp32().items()}
        W_ = Wc.clone().requires_grad_(True)
        b_ = bc.clone().requires_grad_(True)
        with torch.enable_grad():
            x = _forward_with_grad(rp, cfg, ids.numpy(), emulate, features=True)
            nll = torch.nn.functional.cross_entropy(x @ W_.t() + b_, lab.long().cuda(), reduction="none")
            nll.sum().backward()
        gr = {k: (v.grad.detach() if v.grad is not None else torch.zeros_like(v)) for k, v in rp.items()}
        gr["cls_w"], gr["cls_b"] = W_.grad.detach(), b_.grad.detach()
        return gr, nll.detach().cpu().numpy(), x.detach()

    r32, ref_loss, feat32 = ref(False)
    emu, _, _ = ref(True)
    np.testing.assert_allclose(loss.numpy(), ref_loss, rtol=2e-2, atol=2e-3)
    feat = model.features(ids.cuda())
    assert ((feat - feat32).norm() / feat32.norm()).item() < 2e-2
    d = cfg.d_model
    bad, report = [], []
    for name, ref_g in r32.items():
        if name == "cls_w":
            got = tr.hgrad[:C * d].view(C, d)
        elif name == "cls_b":
            got = tr.hgrad[C * d:]
        else:
            got = tr.grad[model.offsets[name]:model.offsets[name] + ref_g.numel()].view(ref_g.shape)
        if name in ("head_w", "head_b"):  # the score head is not part of the classifier
            assert got.abs().max().item() == 0.0
            continue
        e = emu[name]
        if name in ("tok_emb", "pos_emb"):
            used = ref_g.abs().sum(1) > 0
            got, ref_g, e = got[used], ref_g[used], e[used]
        if ref_g.norm() == 0:
            continue
        r_32 = ((got - ref_g).norm() / ref_g.norm()).item()
        floor = ((e - ref_g).norm() / ref_g.norm()).item()
        r_emu = ((got - e).norm() / e.norm()).item()
        report.append((r_32, name, floor, r_emu))
        if not r_32 <= max(2e-2, 1.5 * floor + 2e-3) or not r_emu <= max(2e-2, 2 * floor + 2e-3):
            bad.append(report[-1])
    assert not bad, (bad, sorted(report, reverse=True)[:8])
    assert len(report) > 20


def test_train_classifier_learns():
    from paper_2408_15792_b200.predictors import OptClassifierScorer, train_classifier
    t = _trace(600, seed=7)
    res = train_classifier(t, _cfg(epochs=4), n_buckets=6)
    rep = res.report
    assert rep["kind"] == "classifier" and rep["n_buckets"] == 6 and rep["n_train"] + rep["n_eval"] == 600
    assert rep["steps"] == 4 * len(range(0, 480, 32))
    assert rep["accuracy"] > 0.5 and rep["eval_tau"] > 0.5, rep
    assert isinstance(res.scorer, OptClassifierScorer) and res.scorer.length_calibrated
    s = res.scorer.score_batch(t[:5], seed=0)
    assert all(v % res.scorer.bucket_size == res.scorer.bucket_size / 2.0 for v in s)
    # save / load round trip (the scorer registry, predictors.py:486-527)
    import tempfile, os
    from paper_2408_15792_b200.predictors import load_scorer, save_scorer
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "cls.json")
        save_scorer(res.scorer, path)
        back = load_scorer(path)
        assert isinstance(back, OptClassifierScorer) and back.score_batch(t[:50], 0) == res.scorer.score_batch(t[:50], 0)
    with pytest.raises(ValueError):
        train_classifier(t, _cfg(), n_buckets=1)

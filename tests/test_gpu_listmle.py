"""K6 ListMLE on the B200 vs the reference golden vectors."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_listmle_golden_float64(golden):
    from paper_2408_15792_b200.ranking import list_mle_gradient, list_mle_loss
    for c in golden["listmle_golden"]["cases"]:
        loss = list_mle_loss(c["scores"], c["order"])
        grad = list_mle_gradient(c["scores"], c["order"])
        assert loss == pytest.approx(c["loss"], rel=1e-12, abs=1e-12), c["tag"]
        np.testing.assert_allclose(grad, np.array(c["grad"]), rtol=1e-10, atol=1e-12, err_msg=c["tag"])


def test_listmle_errors_and_degenerate():
    from paper_2408_15792_b200.ranking import list_mle_gradient, list_mle_loss
    with pytest.raises(ValueError):
        list_mle_loss([1.0, 2.0], [0, 0])
    with pytest.raises(ValueError):
        list_mle_gradient([1.0, 2.0, 3.0], [0, 1])
    with pytest.raises(ValueError):
        list_mle_loss([1.0, 2.0], [0, 2])
    assert list_mle_loss([], []) == 0.0
    assert list_mle_loss([3.0], [0]) == 0.0


def test_listmle_training_form_golden(golden):
    from paper_2408_15792_b200.ranking import listmle_from_lengths
    t = golden["listmle_golden"]["train"]
    g = torch.tensor(t["g"], dtype=torch.float32, device="cuda")
    lengths = torch.tensor(t["lengths"], dtype=torch.int32, device="cuda")
    loss, dg = listmle_from_lengths(g, lengths, t["width"])
    # fp32 kernel vs float64 reference on identical fp32 inputs (SURVEY 8c tolerance)
    np.testing.assert_allclose(loss.cpu().numpy(), np.array(t["loss"]), rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(dg.cpu().numpy(), np.array(t["grad"]), atol=1e-5)


@pytest.mark.parametrize("L", [2, 31, 64, 100, 1024])
def test_listmle_training_form_vs_oracle(L):
    from oracle import ranking_oracle as ro
    from paper_2408_15792_b200.ranking import listmle_from_lengths
    rng = np.random.default_rng(L)
    n_lists = 257
    g = rng.normal(0, 3, (n_lists, L)).astype(np.float32)
    lengths = rng.integers(1, 2049, (n_lists, L)).astype(np.int32)
    loss, dg = listmle_from_lengths(torch.from_numpy(g).cuda(), torch.from_numpy(lengths).cuda(), 10)
    want_l, want_g = ro.listmle_train_step_targets(g.astype(np.float64), lengths, 10)
    np.testing.assert_allclose(loss.cpu().numpy(), want_l, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(dg.cpu().numpy(), want_g, atol=1e-5)
    # gradients of each list sum to zero (ranking.py:102-120 property)
    assert np.abs(dg.double().sum(1).cpu().numpy()).max() < 1e-5


def test_listmle_batched_float32_large():
    """1M lists x 64 (the HBM-sweep size) — spot-check a sample against the oracle."""
    from oracle import ranking_oracle as ro
    from paper_2408_15792_b200.ranking import listmle_from_lengths
    gen = torch.Generator(device="cuda").manual_seed(0)
    n_lists, L = 1 << 20, 64
    g = torch.randn(n_lists, L, device="cuda", generator=gen)
    lengths = torch.randint(1, 2049, (n_lists, L), device="cuda", generator=gen, dtype=torch.int32)
    loss, dg = listmle_from_lengths(g, lengths, 10)
    idx = torch.randint(0, n_lists, (64,), generator=torch.Generator().manual_seed(1))
    want_l, want_g = ro.listmle_train_step_targets(g[idx].double().cpu().numpy(), lengths[idx].cpu().numpy(), 10)
    np.testing.assert_allclose(loss[idx].cpu().numpy(), want_l, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(dg[idx].cpu().numpy(), want_g, atol=1e-5)


@pytest.mark.parametrize("case", ["wide_labels", "wide_scores", "ties", "ragged"])
def test_listmle_training_form_register_path_edges(case):
    """L <= 64 runs the register-resident kernel: 64-bit sort keys when labels exceed
    2^25, score ranges far beyond exp's fp32 range, all-equal labels (pure index order)."""
    from oracle import ranking_oracle as ro
    from paper_2408_15792_b200.ranking import listmle_from_lengths
    rng = np.random.default_rng(7)
    n_lists, L, width = 300, 64, 10
    g = rng.normal(0, 3, (n_lists, L)).astype(np.float32)
    lengths = rng.integers(1, 2049, (n_lists, L)).astype(np.int32)
    if case == "wide_labels":
        width = 1
        lengths = rng.integers(-(1 << 31), (1 << 31) - 1, (n_lists, L), dtype=np.int64).astype(np.int32)
    elif case == "wide_scores":
        g = rng.uniform(-1000, 1000, (n_lists, L)).astype(np.float32)
    elif case == "ties":
        lengths[:] = 5
    elif case == "ragged":
        L = 37
        g, lengths = g[:, :L].copy(), lengths[:, :L].copy()
    loss, dg = listmle_from_lengths(torch.from_numpy(g).cuda(), torch.from_numpy(lengths).cuda(), width)
    want_l, want_g = ro.listmle_train_step_targets(g.astype(np.float64), lengths, width)
    # |t| ~ 1000: one fp32 ulp of t (and of t + L) is 6e-5, so the gradient's absolute bar
    # scales with it; everywhere else the standard 1e-5 bar holds
    wide = case == "wide_scores"
    np.testing.assert_allclose(loss.cpu().numpy(), want_l, rtol=1e-5, atol=1e-3 if wide else 1e-6)
    np.testing.assert_allclose(dg.cpu().numpy(), want_g, atol=1e-4 if wide else 1e-5)

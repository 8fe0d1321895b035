"""BASELINE.json configs[0] end to end on the device, against the reference's own run
of the same case (tests/golden/make_cfg1_golden.py): the reference default ranker's
scores for 64 prompts x 128 tokens -> ListMLE (f64, rel 1e-12), one ranking-policy step
(bit-exact batch, promotions and state) and Kendall tau-b (bit-exact counts and tau)."""

import json
import pathlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

G = json.loads((pathlib.Path(__file__).resolve().parent / "golden" / "cfg1_golden.json").read_text())


def test_cfg1_tau_bit_exact():
    from paper_2408_15792_b200.ranking import kendall_tau_b
    r = kendall_tau_b(G["scores"], G["lengths"])
    assert [r.tau, r.concordant, r.discordant, r.n_pairs] == G["tau"]


def test_cfg1_listmle_matches():
    from paper_2408_15792_b200.ranking import bucket_lengths, list_mle_gradient, list_mle_loss
    g = -np.asarray(G["scores"], dtype=np.float64)
    order = np.argsort(np.asarray(bucket_lengths(G["lengths"], 10)), kind="stable")
    assert order.tolist() == G["order"]
    np.testing.assert_allclose(list_mle_loss(g, order), G["listmle_loss"], rtol=1e-12)
    np.testing.assert_allclose(list_mle_gradient(g, order), G["listmle_grad"], rtol=1e-12, atol=1e-14)


def test_cfg1_schedule_bit_exact():
    from paper_2408_15792_b200.schedulers import RankingPolicy, SchedulerConfig
    from paper_2408_15792_b200.workload import Request
    reqs = [Request(id=k, arrival_time=float(k), prompt_tokens=128, true_output_tokens=L, score=s)
            for k, (s, L) in enumerate(zip(G["scores"], G["lengths"]))]
    cfg = SchedulerConfig(max_batch=32, starvation_threshold=100, priority_quantum=50)
    d = RankingPolicy(cfg, G["length_calibrated"]).schedule(reqs, 1 << 62)
    assert (list(d.run), list(d.promoted), list(d.demoted)) == (G["run"], G["promoted"], G["demoted"])
    assert [[r.priority, r.starvation_count, r.quantum] for r in reqs] == G["state"]

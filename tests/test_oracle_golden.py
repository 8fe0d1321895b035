"""The CPU oracle is pinned to golden vectors produced by the reference itself
(tests/golden/make_golden.py, make_large_golden.py). CPU only."""

import math

import numpy as np
import pytest

from oracle import ranking_oracle as ro
from oracle import schedule_oracle as so
from oracle import tau_c


def test_tau_oracle_matches_reference_golden(golden):
    for c in golden["tau_golden"]["cases"]:
        tau, C, D, n0 = ro.kendall_tau_b(c["x"], c["y"])
        assert (C, D, n0) == (c["concordant"], c["discordant"], c["n_pairs"]), c["tag"]
        assert tau == c["tau"], c["tag"]  # same expression on the same ints: bit-equal


def test_tau_c_oracle_matches_reference_golden(golden):
    for c in golden["tau_golden"]["cases"]:
        if len(c["x"]) < 2:
            continue
        C, D, n1, n2, n3 = tau_c.tau_counts(c["x"], c["y"], threads=2)
        assert (C, D) == (c["concordant"], c["discordant"]), c["tag"]
        n0 = len(c["x"]) * (len(c["x"]) - 1) // 2
        denom = math.sqrt((n0 - n1) * (n0 - n2))
        tau = 0.0 if denom == 0.0 else (C - D) / denom
        assert tau == c["tau"], c["tag"]
        assert C + D + n1 + n2 - n3 == n0


def test_tau_c_oracle_matches_large_reference_golden(golden):
    if "large_golden" not in golden:
        pytest.skip("large golden not generated")
    import recipes
    # the 1M pair enumeration takes minutes in C; check the tie counts here (cheap)
    # and leave C/D to the GPU test, which compares against the reference directly.
    for variant, g in golden["large_golden"]["tau"].items():
        x, y = recipes.tau_1m(variant)
        _, cx = np.unique(x.astype(np.float64), return_counts=True)
        _, cy = np.unique(y.astype(np.float64), return_counts=True)
        assert int(np.sum(cx * (cx - 1) // 2)) == g["n1"]
        assert int(np.sum(cy * (cy - 1) // 2)) == g["n2"]


def test_listmle_oracle_matches_reference_golden(golden):
    for c in golden["listmle_golden"]["cases"]:
        assert ro.list_mle_loss(c["scores"], c["order"]) == c["loss"], c["tag"]
        np.testing.assert_array_equal(ro.list_mle_gradient(c["scores"], c["order"]), np.array(c["grad"]))
    t = golden["listmle_golden"]["train"]
    loss, grad = ro.listmle_train_step_targets(np.array(t["g"], dtype=np.float32).astype(np.float64),
                                               np.array(t["lengths"]), t["width"])
    np.testing.assert_array_equal(loss, np.array(t["loss"]))
    np.testing.assert_array_equal(grad, np.array(t["grad"]))


def test_listmle_oracle_errors():
    with pytest.raises(ValueError):
        ro.list_mle_loss([1.0, 2.0], [0, 0])
    with pytest.raises(ValueError):
        ro.bucket_lengths([1], 0)
    assert ro.bucket_lengths([0, 9, 10, 19, 20], 10).tolist() == [0, 0, 1, 1, 2]


class _R:
    def __init__(self, **kw):
        self.__dict__.update(kw)


def schedule_requests(init):
    rs = []
    for k in range(len(init["id"])):
        rs.append(_R(id=init["id"][k], arrival_time=init["arrival"][k], prompt_tokens=init["prompt"][k],
                     generated_tokens=init["generated"][k], score=init["score"][k],
                     state="running" if init["running"][k] else "waiting", priority=init["priority"][k],
                     starvation_count=init["starvation"][k], quantum=init["quantum"][k]))
    return rs


def test_schedule_oracle_matches_reference_golden(golden):
    for case in golden["schedule_golden"]["cases"]:
        cfg = case["config"]
        reqs = schedule_requests(case["init"])
        kv = (1 << 62) if case["kv_budget"] is None else case["kv_budget"]
        for step in case["steps"]:
            run, prom, dem = so.schedule(reqs, kv, max_batch=cfg["max_batch"], preemption=cfg["preemption"],
                                         threshold=cfg["starvation_threshold"], quantum=cfg["priority_quantum"],
                                         calibrated=case["calibrated"])
            assert (run, prom, dem) == (step["run"], step["promoted"], step["demoted"])
            assert [bool(r.priority) for r in reqs] == step["state"]["priority"]
            assert [r.starvation_count for r in reqs] == step["state"]["starvation"]
            assert [r.quantum for r in reqs] == step["state"]["quantum"]

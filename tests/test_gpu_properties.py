"""The reference's property tests (test_ranking.py:72-90, :119-175; hypothesis) run
against the device implementations, with the exact C / numpy oracle as the referee
where the reference's test compares to a brute force."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

pytestmark = pytest.mark.gpu


@given(st.lists(st.integers(0, 4), min_size=2, max_size=25))
@settings(max_examples=60, deadline=None)
def test_tau_self_correlation_property(xs):
    from paper_2408_15792_b200.ranking import kendall_tau_b
    t = kendall_tau_b(xs, xs).tau
    if len(set(xs)) > 1:
        assert t == pytest.approx(1.0)
    else:
        assert t == 0.0


@given(st.lists(st.floats(-50, 50, allow_nan=False), min_size=2, max_size=25),
       st.lists(st.floats(-50, 50, allow_nan=False), min_size=2, max_size=25))
@settings(max_examples=60, deadline=None)
def test_tau_bounds_antisymmetry_and_oracle(xs, ys):
    from oracle import ranking_oracle as ro
    from paper_2408_15792_b200.ranking import kendall_tau_b
    n = min(len(xs), len(ys))
    xs, ys = xs[:n], ys[:n]
    r = kendall_tau_b(xs, ys)
    assert -1.0 - 1e-12 <= r.tau <= 1.0 + 1e-12
    assert kendall_tau_b([-v for v in xs], ys).tau == pytest.approx(-r.tau, abs=1e-12)
    assert (r.tau, r.concordant, r.discordant, r.n_pairs) == ro.kendall_tau_b(xs, ys)


@given(st.lists(st.floats(-20, 20, allow_nan=False), min_size=1, max_size=40), st.floats(-100, 100),
       st.randoms(use_true_random=False))
@settings(max_examples=60, deadline=None)
def test_listmle_shift_invariance_and_zero_sum(scores, shift, rnd):
    from paper_2408_15792_b200.ranking import list_mle_gradient, list_mle_loss
    s = np.asarray(scores, dtype=np.float64)
    order = np.arange(len(s))
    rnd.shuffle(order)
    base = list_mle_loss(s, order)
    assert list_mle_loss(s + shift, order) == pytest.approx(base, rel=1e-10, abs=1e-10)
    g = list_mle_gradient(s, order)
    assert abs(float(np.sum(g))) < 1e-9


@given(st.lists(st.floats(-5, 5, allow_nan=False), min_size=2, max_size=20), st.randoms(use_true_random=False))
@settings(max_examples=40, deadline=None)
def test_listmle_margin_monotonicity(scores, rnd):
    """test_ranking.py:119-124: raising the score of the target's first item lowers the loss."""
    from paper_2408_15792_b200.ranking import list_mle_loss
    s = np.asarray(scores, dtype=np.float64)
    order = np.arange(len(s))
    rnd.shuffle(order)
    hi = s.copy()
    hi[order[0]] += 1.0
    assert list_mle_loss(hi, order) < list_mle_loss(s, order) + 1e-12

"""CPU restatement of ranksched.ranking — TEST INFRASTRUCTURE ONLY (checker, never shipped).

Each function follows the reference line by line in float64 numpy:
  kendall_tau_b        ranking.py:24-63   (O(n^2) row loop of sign products + np.unique ties)
  list_mle_loss        ranking.py:86-99   (reversed logaddexp.accumulate suffix LSE)
  list_mle_gradient    ranking.py:102-120 (forward logaddexp.accumulate of -lse)
  bucket_lengths       ranking.py:123-132
and tau_counts() additionally returns the tie counts n1, n2, n3 the B200 kernel
exposes (n3 = pairs tied in both coordinates, by direct enumeration of the pair
products like the row loop).
"""

from __future__ import annotations

import math

import numpy as np


def tau_counts(x, y):
    """(C, D, n1, n2, n3) by the reference row loop (ranking.py:45-57)."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if x.shape != y.shape or x.ndim != 1:
        raise ValueError("kendall_tau_b expects two equal-length 1-d arrays")
    n = len(x)
    c = d = n3 = 0
    for i in range(n - 1):
        dx = np.sign(x[i + 1:] - x[i])
        dy = np.sign(y[i + 1:] - y[i])
        prod = dx * dy
        c += int(np.count_nonzero(prod > 0))
        d += int(np.count_nonzero(prod < 0))
        n3 += int(np.count_nonzero((dx == 0) & (dy == 0)))

    def tied_pairs(v):
        _, counts = np.unique(v, return_counts=True)
        return int(np.sum(counts * (counts - 1) // 2))

    return c, d, tied_pairs(x) if n else 0, tied_pairs(y) if n else 0, n3


def kendall_tau_b(x, y):
    """Returns (tau, C, D, n0) exactly like ranking.py:24-63."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if x.shape != y.shape or x.ndim != 1:
        raise ValueError("kendall_tau_b expects two equal-length 1-d arrays")
    n = len(x)
    n0 = n * (n - 1) // 2
    if n0 == 0:
        return 0.0, 0, 0, 0
    c, d, n1, n2, _ = tau_counts(x, y)
    denom = math.sqrt((n0 - n1) * (n0 - n2))
    if denom == 0.0:
        return 0.0, c, d, n0
    return (c - d) / denom, c, d, n0


def _check(scores, true_order):
    scores = np.asarray(scores, dtype=np.float64)
    order = np.asarray(true_order, dtype=np.int64)
    if scores.ndim != 1 or order.shape != scores.shape:
        raise ValueError("scores and true_order must be equal-length 1-d arrays")
    if len(order) and (np.sort(order) != np.arange(len(order))).any():
        raise ValueError("true_order must be a permutation of 0..n-1")
    return scores, order


def _suffix_lse(t):
    return np.logaddexp.accumulate(t[::-1])[::-1]


def list_mle_loss(scores, true_order) -> float:
    scores, order = _check(scores, true_order)
    if len(scores) == 0:
        return 0.0
    t = scores[order]
    return float(np.sum(_suffix_lse(t) - t))


def list_mle_gradient(scores, true_order) -> np.ndarray:
    scores, order = _check(scores, true_order)
    n = len(scores)
    grad = np.zeros(n)
    if n == 0:
        return grad
    t = scores[order]
    lse = _suffix_lse(t)
    L = np.logaddexp.accumulate(-lse)
    grad[order] = np.exp(t + L) - 1.0
    return grad


def bucket_lengths(lengths, bucket_width: int = 10) -> np.ndarray:
    if bucket_width < 1:
        raise ValueError("bucket_width must be >= 1")
    return np.asarray(lengths, dtype=np.int64) // bucket_width


def listmle_train_step_targets(g, lengths, bucket_width=10):
    """The per-list quantities of predictors.py:379-384 for a batch of lists:
    loss/n and grad/n with order = stable argsort of bucketed lengths."""
    g = np.asarray(g, dtype=np.float64)
    lengths = np.asarray(lengths)
    losses = np.empty(g.shape[0])
    grads = np.empty_like(g)
    n = g.shape[1]
    for k in range(g.shape[0]):
        order = np.argsort(bucket_lengths(lengths[k], bucket_width), kind="stable")
        losses[k] = list_mle_loss(g[k], order) / n
        grads[k] = list_mle_gradient(g[k], order) / n
    return losses, grads

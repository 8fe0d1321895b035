"""Seeded input recipes shared by the golden generators and the tests (no reference
imports here: the GPU box regenerates the inputs from these recipes)."""

from __future__ import annotations

import numpy as np


def tau_1m(variant: str = "f32", n: int = 1_000_000):
    """cfg4 (BASELINE.json configs[3]): scores fp32 N(0,1) with -0.0 injected at 1%,
    true lengths uniform int [1, 2048]; variant 'bf16' rounds scores to bf16 (heavy ties)."""
    rng = np.random.default_rng(4)
    x = rng.normal(size=n).astype(np.float32)
    y = rng.integers(1, 2049, n).astype(np.int32)
    zero = rng.random(n) < 0.01
    x[zero] = np.float32(-0.0)
    if variant == "bf16":
        b = x.view(np.uint32)
        b = ((b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)  # round-to-nearest-even
        x = b.view(np.float32)
    return x, y


def queue_1m(n: int = 1_000_000, shuffled_ids: bool = False):
    """cfg4 queue: Poisson(40/s) arrivals in order, ids in arrival order (or shuffled),
    fp32 scores N(0,1) as float64, 1% priority with quantum U[0,50], starvation U[0,100),
    prompt tokens U[1,1024], generated U[0,200], 30% running."""
    rng = np.random.default_rng(4)
    arrival = np.cumsum(rng.exponential(1 / 40.0, n))
    ids = np.arange(n, dtype=np.int64)
    if shuffled_ids:
        ids = rng.permutation(n).astype(np.int64)
    score = rng.normal(size=n).astype(np.float32).astype(np.float64)
    priority = rng.random(n) < 0.01
    quantum = np.where(priority, rng.integers(0, 51, n), 0).astype(np.int32)
    starvation = rng.integers(0, 100, n).astype(np.int32)
    prompt = rng.integers(1, 1025, n).astype(np.int32)
    generated = rng.integers(0, 201, n).astype(np.int32)
    running = rng.random(n) < 0.3
    return dict(arrival=arrival, ids=ids, score=score, priority=priority, quantum=quantum,
                starvation=starvation, prompt=prompt, generated=generated, running=running)

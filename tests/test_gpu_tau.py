"""K10 tau counts on the B200 vs the reference (golden vectors) — bit-exact C, D, tau."""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_tau_golden_bit_exact(golden):
    from paper_2408_15792_b200.ranking import kendall_tau_b
    for c in golden["tau_golden"]["cases"]:
        r = kendall_tau_b(c["x"], c["y"])
        assert (r.concordant, r.discordant, r.n_pairs) == (c["concordant"], c["discordant"], c["n_pairs"]), c["tag"]
        assert r.tau == c["tau"], c["tag"]


@pytest.mark.parametrize("xdt", [np.float32, np.float64, np.int32, np.int64])
@pytest.mark.parametrize("ydt", [np.float32, np.float64, np.int32, np.int64])
def test_tau_dtypes_agree_with_oracle(xdt, ydt):
    from oracle import tau_c
    from paper_2408_15792_b200.ranking import kendall_tau_b
    rng = np.random.default_rng(17)
    n = 5000
    x = rng.integers(-50, 50, n).astype(xdt)
    y = rng.integers(0, 30, n).astype(ydt)
    r = kendall_tau_b(x, y)
    C, D, n1, n2, _ = tau_c.tau_counts(x, y)
    assert (r.concordant, r.discordant) == (C, D)
    n0 = n * (n - 1) // 2
    assert r.tau == (C - D) / math.sqrt((n0 - n1) * (n0 - n2))


def test_tau_float64_precision_semantics():
    # int64 values that collide once cast to float64 must tie (np.asarray(..., float64))
    from paper_2408_15792_b200.ranking import kendall_tau_b
    from oracle import ranking_oracle as ro
    big = 2 ** 53
    x = np.array([big, big + 1, big + 2, 5, -3], dtype=np.int64)
    y = np.array([1, 2, 3, 4, 5], dtype=np.int64)
    r = kendall_tau_b(x, y)
    assert (r.tau, r.concordant, r.discordant, r.n_pairs) == ro.kendall_tau_b(x, y)


def test_tau_rejects_bad_input():
    from paper_2408_15792_b200.ranking import kendall_tau_b
    with pytest.raises(ValueError):
        kendall_tau_b([1, 2], [1, 2, 3])
    assert kendall_tau_b([], []).tau == 0.0


def test_tau_nan_like_reference(ranksched):
    """NaN pairs count as neither concordant nor discordant and NaNs tie with each other
    (np.unique equal_nan), exactly as the reference's row loop (ranking.py:45-57)."""
    from paper_2408_15792_b200.ranking import kendall_tau_b
    rng = np.random.default_rng(23)
    cases = [([1.0, float("nan"), 2.0], [1, 2, 3]), ([float("nan")] * 4, [1, 2, 3, 4]),
             ([1.0, 2.0, 3.0], [float("nan"), 1.0, float("nan")]), ([np.inf, np.inf, -np.inf, np.nan], [1, 2, 3, 4])]
    for n in (50, 2000):
        x = rng.normal(size=n)
        y = rng.integers(0, 20, n).astype(np.float64)
        x[rng.random(n) < 0.1] = np.nan
        y[rng.random(n) < 0.05] = np.nan
        cases.append((x, y))
        cases.append((x.astype(np.float32), rng.integers(0, 9, n)))
    for x, y in cases:
        want = ranksched.ranking.kendall_tau_b(x, y)
        r = kendall_tau_b(x, y)
        assert (r.tau, r.concordant, r.discordant, r.n_pairs) == \
            (want.tau, want.concordant, want.discordant, want.n_pairs)


def test_tau_1m_matches_reference(golden):
    import recipes
    from paper_2408_15792_b200.ranking import kendall_tau_b
    if "large_golden" not in golden:
        pytest.skip("large golden not generated")
    for variant, g in golden["large_golden"]["tau"].items():
        x, y = recipes.tau_1m(variant)
        r = kendall_tau_b(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
        assert (r.concordant, r.discordant) == (g["concordant"], g["discordant"]), variant
        n0 = g["n"] * (g["n"] - 1) // 2
        assert r.tau == (g["concordant"] - g["discordant"]) / math.sqrt((n0 - g["n1"]) * (n0 - g["n2"]))


def test_tau_large_n_properties():
    """Size-independent identities at 16M: tau(x, x) = 1 with ties excluded, antisymmetry,
    permutation invariance, and C + D + n1 + n2 - n3 = n0."""
    from paper_2408_15792_b200.ranking import tau_counts_device
    g = torch.Generator(device="cuda").manual_seed(3)
    n = 1 << 24
    x = torch.randn(n, device="cuda", generator=g)
    y = torch.randint(1, 2049, (n,), device="cuda", generator=g, dtype=torch.int32)
    c = tau_counts_device(x, y).cpu().tolist()
    n0 = n * (n - 1) // 2
    C, D, n1, n2, n3, nan = c
    assert nan == 0 and C + D + n1 + n2 - n3 == n0
    cm = tau_counts_device(-x, y).cpu().tolist()
    assert (cm[0], cm[1]) == (D, C)
    perm = torch.randperm(n, device="cuda", generator=g)
    cp = tau_counts_device(x[perm].contiguous(), y[perm].contiguous()).cpu().tolist()
    assert cp[:5] == c[:5]
    cs = tau_counts_device(y, y).cpu().tolist()
    assert cs[1] == 0 and cs[0] == n0 - cs[2]


def test_tau_plan_graph_matches_eager():
    """TauPlan (the kernels captured as one CUDA graph) gives the eager counts, and
    replays track input updates made in place."""
    import torch
    from paper_2408_15792_b200 import ranking
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(300_000, device="cuda", generator=g)
    y = torch.randint(1, 2049, (300_000,), device="cuda", generator=g, dtype=torch.int32)
    plan = ranking.TauPlan(x, y)
    want = ranking.tau_counts_device(x, y).clone()
    assert torch.equal(plan(), want)
    x.copy_(torch.randn(300_000, device="cuda", generator=g))
    want2 = ranking.tau_counts_device(x, y).clone()
    assert torch.equal(plan(), want2) and not torch.equal(want, want2)


@pytest.mark.parametrize("y_span", [4095, 4096, "float"])
def test_tau_histogram_and_merge_paths_vs_oracle(y_span):
    """y images spanning < 4096 values take the histogram path for cross-tile
    inversions, wider ones the merge passes; both exact against the pair-loop oracle."""
    from oracle import tau_c
    from paper_2408_15792_b200.ranking import kendall_tau_b
    rng = np.random.default_rng(23)
    n = 40_000
    x = rng.integers(-3000, 3000, n).astype(np.float32)
    if y_span == "float":
        y = rng.normal(size=n).astype(np.float32)
    else:
        y = rng.integers(0, y_span + 1, n).astype(np.int32) + 7
        y[:2] = (7, 7 + y_span)  # pin the span
    r = kendall_tau_b(x, y)
    C, D, n1, n2, _ = tau_c.tau_counts(x, y)
    assert (r.concordant, r.discordant) == (C, D)
    n0 = n * (n - 1) // 2
    assert r.tau == (C - D) / math.sqrt((n0 - n1) * (n0 - n2))


def test_tau_paths_agree_at_16m():
    """The same ranks of y, once spanning 2048 values (histogram path) and once scaled to
    span 2e8 (merge path), give identical counts at 16M (several tiles per chunk)."""
    from paper_2408_15792_b200.ranking import tau_counts_device
    g = torch.Generator(device="cuda").manual_seed(9)
    n = 1 << 24
    x = torch.randn(n, device="cuda", generator=g).to(torch.bfloat16).float()  # heavy x ties
    y = torch.randint(1, 2049, (n,), device="cuda", generator=g, dtype=torch.int32)
    a = tau_counts_device(x, y).cpu().tolist()
    b = tau_counts_device(x, y * 100_000).cpu().tolist()
    assert a == b


def _fast_cases(rng):
    """Inputs that drive every branch of the bucket fast path (tau_fast.cu)."""
    n = 60_000
    yl = rng.integers(1, 2049, n).astype(np.int32)
    near1 = (1.0 + 1e-4 * rng.normal(size=n)).astype(np.float32)  # few top-bit buckets -> level-2 splits
    one = np.float32(1.0).view(np.int32)
    crowd2 = np.where(rng.random(n) < 0.5, one, one + 1).view(np.float32)  # two adjacent images
    crowd2[:2] = (-1e30, 1e30)  # full range: the level-2 child keeps 8 x bits, > cap keys
    crowd40 = (one + rng.integers(0, 40, n).astype(np.int32)).view(np.float32)  # 40 adjacent images
    crowd40[:2] = (-1e30, 1e30)  # > 16 distinct x in one crowded child -> general path
    return {
        "normal": (rng.normal(size=n).astype(np.float32), yl),
        "bf16_ties": (torch.from_numpy(rng.normal(size=n).astype(np.float32)).bfloat16().float().numpy(), yl),
        "near_one_split": (near1, yl),
        "small_int_x": (rng.integers(-40, 40, n).astype(np.int32), yl),  # single-x buckets
        "all_x_equal": (np.full(n, 3.5, np.float32), yl),
        "all_y_equal": (rng.normal(size=n).astype(np.float32), np.full(n, 7, np.int32)),
        "huge_single": (np.where(rng.random(n) < 0.9, 0.25, rng.normal(size=n)).astype(np.float32), yl),
        "crowded_two_values": (crowd2, yl),
        "crowded_child_fallback": (crowd40, yl),
        "f64_x_i64_y": (rng.normal(size=n), rng.integers(0, 3000, n).astype(np.int64)),
        "neg_zero": (np.where(rng.random(n) < 0.3, -0.0, rng.normal(size=n)).astype(np.float32), yl),
        "tiny": (np.array([2.0, 1.0, 2.0], np.float32), np.array([1, 2, 1], np.int32)),
    }


@pytest.mark.parametrize("case", ["normal", "bf16_ties", "near_one_split", "small_int_x", "all_x_equal",
                                  "all_y_equal", "huge_single", "crowded_two_values", "crowded_child_fallback", "f64_x_i64_y",
                                  "neg_zero", "tiny"])
def test_tau_fast_path_vs_oracle(case, monkeypatch):
    """The bucket fast path (and its fallback) against the exhaustive pair oracle:
    C, D, n1, n2, n3 bit-exact (RS_TAU_PATH=fast: these sizes are below the crossover
    where rs_tau_counts picks the fast path by itself)."""
    monkeypatch.setenv("RS_TAU_PATH", "fast")
    from oracle import tau_c
    from paper_2408_15792_b200.ranking import tau_counts_device
    x, y = _fast_cases(np.random.default_rng(41))[case]
    got = tau_counts_device(torch.from_numpy(np.ascontiguousarray(x)).cuda(),
                            torch.from_numpy(np.ascontiguousarray(y)).cuda()).cpu().tolist()
    want = list(tau_c.tau_counts(x, y))
    assert got[:5] == want and got[5] == 0, (case, got, want)
    fast = tau_counts_device(torch.from_numpy(np.ascontiguousarray(x)).cuda(),
                             torch.from_numpy(np.ascontiguousarray(y)).cuda(), fast_only=True).cpu().tolist()
    if case == "crowded_child_fallback":
        assert fast[5] == 2  # the fast path declines; rs_tau_counts ran the general path
    else:
        assert fast == got


def test_tau_plan_counts_falls_back(monkeypatch):
    """TauPlan replays the fast path only; counts() runs the general path when y is wide."""
    monkeypatch.setenv("RS_TAU_PATH", "fast")
    from paper_2408_15792_b200 import ranking
    g = torch.Generator(device="cuda").manual_seed(6)
    x = torch.randn(200_000, device="cuda", generator=g)
    y = torch.randn(200_000, device="cuda", generator=g)  # wide y: general path
    plan = ranking.TauPlan(x, y)
    assert int(plan()[5]) == 2
    assert torch.equal(plan.counts(), ranking.tau_counts_device(x, y))


@pytest.mark.parametrize("n", [1 << 20, 1 << 26])
def test_tau_fast_equals_general_large(n, monkeypatch):
    """At sizes with level-2 splits over many chunks, the fast path equals the general
    path on the same inputs (forced by RS_TAU_PATH) and on the same ranks with y scaled past
    the 4096-value window."""
    from paper_2408_15792_b200.ranking import tau_counts_device
    g = torch.Generator(device="cuda").manual_seed(n & 0xffff)
    x = torch.randn(n, device="cuda", generator=g)
    y = torch.randint(1, 2049, (n,), device="cuda", generator=g, dtype=torch.int32)
    monkeypatch.setenv("RS_TAU_PATH", "fast")
    a = tau_counts_device(x, y, fast_only=True).cpu().tolist()
    monkeypatch.setenv("RS_TAU_PATH", "general")
    b = tau_counts_device(x, y).cpu().tolist()
    monkeypatch.delenv("RS_TAU_PATH")
    c = tau_counts_device(x, y * 100_000).cpu().tolist()
    assert a[5] == 0 and a == b and a[:2] == c[:2] and a[4] == c[4]

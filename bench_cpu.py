"""CPU baselines timed beside the B200 path on the box's own host cores ("the
reference CPU path is timed on the box's own host cores in the same run").

Test / measurement infrastructure, like oracle/: only bench.py imports this module.
Where the reference has the code (everything but the OPT backbone) the baseline is the
UNMODIFIED reference package staged under oracle/_ref (`kind: "reference"`); the OPT-125M
forward / backward, which the reference does not have, is the torch fp32 restatement in
oracle/opt_ranker.py on all host threads (`kind: "port"`). Every function times a bounded
sample of the named workload and says what the sample was.
"""

from __future__ import annotations

import os
import pathlib
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
for _p in (str(ROOT), str(ROOT / "tests" / "golden")):
    if _p not in sys.path:
        sys.path.insert(0, _p)


def cores() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def reference():
    """The staged reference package, or None (then the oracle port stands in)."""
    try:
        from oracle import install_ref
        return install_ref.import_ranksched()
    except ImportError:
        return None


def _best(fn, reps):
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    return best


# ---------------------------------------------------------------------------
# headline (cfg2): OPT-125M-shape scoring + score sort
# ---------------------------------------------------------------------------


class HeadlineCPU:
    """fp32 OPT forward (oracle port, torch CPU on all threads) on a sample of prompts +
    the reference's RankingPolicy.schedule over those prompts (max_batch 256)."""

    def __init__(self, cfg, S, n_prompts):
        import torch
        from paper_2408_15792_b200.ranker import init_params
        self.torch = torch
        torch.set_num_threads(cores())
        self.cfg, self.S, self.n = cfg, S, n_prompts
        self.params = {k: v.to(torch.bfloat16).float() for k, v in init_params(cfg, 0).items()}
        self.ids = np.random.default_rng(1).integers(4, cfg.vocab, (n_prompts, S)).astype(np.int32)
        self.rs = reference()

    def step(self):
        from oracle import opt_ranker
        g = opt_ranker.forward(self.params, self.cfg, self.ids).numpy()
        if self.rs is not None:
            W = self.rs.workload
            reqs = [W.Request(id=k, arrival_time=float(k), prompt_tokens=self.S, true_output_tokens=1, prompt="")
                    for k in range(len(g))]
            for r, v in zip(reqs, g):
                r.score = -float(v)
            S = self.rs.schedulers
            S.RankingPolicy(S.SchedulerConfig(max_batch=256, starvation_threshold=100, priority_quantum=50),
                            False).schedule(reqs, 1 << 62)
        else:
            from oracle import schedule_oracle

            class R:
                __slots__ = ("id", "arrival_time", "prompt_tokens", "generated_tokens", "score", "state",
                             "priority", "starvation_count", "quantum")
            reqs = []
            for k, v in enumerate(g):
                r = R()
                r.id, r.arrival_time, r.prompt_tokens, r.generated_tokens = k, float(k), self.S, 0
                r.score, r.state, r.priority, r.starvation_count, r.quantum = -float(v), "waiting", False, 0, 0
                reqs.append(r)
            schedule_oracle.schedule(reqs, 1 << 62, max_batch=256, threshold=100, quantum=50, calibrated=False)
        return g

    @property
    def kind(self):
        return "port"

    def describe(self, dt):
        sched = "reference RankingPolicy.schedule" if self.rs is not None else "oracle ranking step"
        return (f"{self.n} prompts x {self.S} tokens per step: oracle fp32 OPT-125M-shape forward (torch CPU, "
                f"{self.torch.get_num_threads()} threads; the reference has no OPT model) + {sched}; {dt:.2f} s/step")


def headline(cfg, S, n_prompts=16, reps=2):
    h = HeadlineCPU(cfg, S, n_prompts)
    h.params_warm = h.step()  # warm-up (allocator, thread pool)
    dt = _best(h.step, reps)
    return {"value": n_prompts / dt, "unit": "prompts/s", "cores": h.torch.get_num_threads(), "kind": h.kind,
            "sample": h.describe(dt)}


def linear_scorer(n_prompts=1024, S=512):
    """The reference's default ranker (featurize + standardised linear model trained with
    the desk_burst recipe, predictors.py:228-259) scoring prompts of S tokens: a DIFFERENT
    model than the OPT ranker, reported for scale only."""
    rs = reference()
    if rs is None:
        return None
    W, P = rs.workload, rs.predictors
    scorer = P.train_ranking(W.generate_burst(2000, W.LengthDist.parse("lognormal(5.0,0.8)"), seed=11,
                                              prompt_noise=0.25), P.TrainConfig(seed=0)).scorer
    rng = np.random.default_rng(0)
    prompts = [" ".join(W._VOCAB[i] for i in rng.integers(0, len(W._VOCAB), S)) for _ in range(n_prompts)]

    def run():
        reqs = [W.Request(id=k, arrival_time=0.0, prompt_tokens=S, true_output_tokens=1, prompt=p)
                for k, p in enumerate(prompts)]  # featurize runs in Request.__post_init__
        scorer.score_batch(reqs, 0)

    dt = _best(run, 1)
    return {"value": n_prompts / dt, "unit": "prompts/s", "cores": 1, "kind": "reference",
            "sample": f"{n_prompts} prompts x {S} tokens: reference featurize + RankingModelScorer.score_batch "
                      f"(linear model, desk_burst recipe) — a different model than the OPT ranker; {dt:.2f} s"}


# ---------------------------------------------------------------------------
# cfg4: tau and the rank step
# ---------------------------------------------------------------------------


def tau(n_sample=32768, n_scipy=1_000_000):
    import recipes
    x, y = recipes.tau_1m("f32")
    rs = reference()
    xs, ys = x[:n_sample], y[:n_sample]
    if rs is not None:
        fn, kind, who = rs.ranking.kendall_tau_b, "reference", "reference kendall_tau_b (ranking.py:24-63)"
    else:
        from oracle import ranking_oracle
        fn, kind, who = ranking_oracle.kendall_tau_b, "port", "oracle restatement of kendall_tau_b"
    dt = _best(lambda: fn(xs, ys), 1)
    pairs = n_sample * (n_sample - 1) / 2
    out = {"value": pairs / dt, "unit": "pairs/s", "cores": 1, "kind": kind,
           "sample": f"{who} on the first {n_sample} rows of the cfg4 1M (x, y): {dt:.2f} s; the O(n^2) row loop "
                     f"at 1M would take ~{dt * (1e6 / n_sample) ** 2 / 60:.0f} min"}
    try:
        from scipy import stats
        ts = _best(lambda: stats.kendalltau(x[:n_scipy], y[:n_scipy]), 1)
        out["scipy_comparator"] = {"value": n_scipy * (n_scipy - 1) / 2 / ts, "unit": "pairs/s", "seconds": ts,
                                   "n": n_scipy, "note": "scipy.stats.kendalltau (O(n log n), not the reference)"}
    except ImportError:
        pass
    return out


def rank_step(n_sample=262144):
    import recipes
    q = recipes.queue_1m(n_sample)
    rs = reference()
    if rs is None:
        return None
    W, S = rs.workload, rs.schedulers
    RUN = W.RequestState.RUNNING
    reqs = []
    for k in range(n_sample):
        r = W.Request(id=int(q["ids"][k]), arrival_time=float(q["arrival"][k]), prompt_tokens=int(q["prompt"][k]),
                      true_output_tokens=1, prompt="", features=np.zeros(0))
        r.score, r.priority = float(q["score"][k]), bool(q["priority"][k])
        r.quantum, r.starvation_count = int(q["quantum"][k]), int(q["starvation"][k])
        r.generated_tokens = int(q["generated"][k])
        if q["running"][k]:
            r.state = RUN
        reqs.append(r)
    pol = S.RankingPolicy(S.SchedulerConfig(max_batch=256, starvation_threshold=100, priority_quantum=50), False)
    dt = _best(lambda: pol.schedule(reqs, 1 << 62), 1)
    return {"value": n_sample / dt, "unit": "requests/s", "cores": 1, "kind": "reference",
            "sample": f"reference RankingPolicy.schedule (schedulers.py:219-240) over the first {n_sample} rows of "
                      f"the cfg4 queue: {dt:.2f} s"}


def listmle(n_lists=1024, L=64):
    """The reference's train_ranking inner ListMLE (predictors.py:379-384) over n_lists."""
    rs = reference()
    if rs is None:
        return None
    R = rs.ranking
    rng = np.random.default_rng(0)
    g = rng.normal(size=(n_lists, L))
    lengths = rng.integers(1, 2049, (n_lists, L))

    def run():
        for gl, yl in zip(g, lengths):
            order = np.argsort(R.bucket_lengths(yl, 10), kind="stable")
            R.list_mle_loss(gl, order)
            R.list_mle_gradient(gl, order)

    dt = _best(run, 3)
    return {"value": n_lists * L / dt, "unit": "items/s", "cores": 1, "kind": "reference",
            "sample": f"reference bucket_lengths + stable argsort + list_mle_loss + list_mle_gradient over "
                      f"{n_lists} lists x {L}: {dt * 1e3:.1f} ms"}


# ---------------------------------------------------------------------------
# cfg3: training step
# ---------------------------------------------------------------------------


def train_step(cfg, S=128, list_len=16):
    """fp32 OPT fwd + ListMLE + backward (oracle port with torch autograd, all threads)
    on one list; the reference has no OPT model (its train_ranking trains the linear
    net). prompts/s of one list of `list_len` prompts."""
    import torch
    from oracle import opt_ranker
    from paper_2408_15792_b200.ranker import init_params
    torch.set_num_threads(cores())
    params = {k: v.to(torch.bfloat16).float().requires_grad_(True) for k, v in init_params(cfg, 0).items()}
    rng = np.random.default_rng(2)
    ids = rng.integers(4, cfg.vocab, (list_len, S))
    lengths = rng.integers(1, 2049, (1, list_len))

    def run():
        for p in params.values():
            p.grad = None
        g = opt_ranker.forward_grad(params, cfg, ids)
        opt_ranker.listmle_torch(g.view(1, list_len), lengths).backward()

    run()
    dt = _best(run, 1)
    return {"value": list_len / dt, "unit": "prompts/s", "cores": torch.get_num_threads(), "kind": "port",
            "sample": f"one list of {list_len} prompts x {S} tokens: oracle fp32 OPT-125M-shape forward + ListMLE + "
                      f"autograd backward (torch CPU); {dt:.2f} s (no optimizer step)"}


# ---------------------------------------------------------------------------
# cfg5: end-to-end loop
# ---------------------------------------------------------------------------


def engine_loop(trace, n_prefix=2000):
    """The reference's engine.run (engine.py:382-460) with its default trained ranker
    (the linear desk_burst model: the reference has no OPT) on the first n_prefix requests
    of the cfg5 trace, max_batch 256, starvation 100 / 50, default cost preset."""
    rs = reference()
    if rs is None:
        return None
    W, P, E, S = rs.workload, rs.predictors, rs.engine, rs.schedulers
    scorer = P.train_ranking(W.generate_burst(2000, W.LengthDist.parse("lognormal(5.0,0.8)"), seed=11,
                                              prompt_noise=0.25), P.TrainConfig(seed=0)).scorer
    reqs = [W.Request(id=r.id, arrival_time=r.arrival_time, prompt_tokens=r.prompt_tokens,
                      true_output_tokens=r.true_output_tokens, prompt=r.prompt) for r in list(trace)[:n_prefix]]
    tr = W.Trace(reqs, {"name": "prefix", "n": n_prefix})
    sched = S.SchedulerConfig(max_batch=256, starvation_threshold=100, priority_quantum=50)
    t0 = time.perf_counter()
    res = E.run(tr, "ranking", scorer, sched=sched)
    dt = time.perf_counter() - t0
    return {"value": n_prefix / dt, "unit": "requests/s", "cores": 1, "kind": "reference",
            "sample": f"reference engine.run(trace[:{n_prefix}], 'ranking', linear desk_burst scorer): {dt:.1f} s, "
                      f"{len(res.records)} steps"}

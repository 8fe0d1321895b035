"""BASELINE.json configs[0] recorded from the reference itself, as the
parity fixture of the whole CPU-runnable case: the reference's default ranker (linear
ListMLE model trained with the desk_burst recipe) scores 64 synthetic prompts of 128
whitespace tokens; then ListMLE(-scores, stable order of len // 10), one
RankingPolicy.schedule step (max_batch 32, threshold 100, quantum 50) and
kendall_tau_b(scores, lengths). Run in the build container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_cfg1_golden.py
"""

from __future__ import annotations

import json
import pathlib
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from ranksched import ranking  # noqa: E402
from ranksched.predictors import TrainConfig, train_ranking  # noqa: E402
from ranksched.schedulers import RankingPolicy, SchedulerConfig  # noqa: E402
from ranksched.workload import _VOCAB, LengthDist, Request, generate_burst  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parent / "cfg1_golden.json"


def main():
    rng = np.random.default_rng(0)
    n, toks = 64, 128
    prompts = [" ".join(_VOCAB[i] for i in rng.integers(0, len(_VOCAB), toks)) for _ in range(n)]
    lengths = rng.integers(1, 2049, n)
    reqs = [Request(id=k, arrival_time=float(k), prompt_tokens=toks, true_output_tokens=int(lengths[k]),
                    prompt=prompts[k]) for k in range(n)]
    train = generate_burst(2000, LengthDist.parse("lognormal(5.0,0.8)"), seed=11, prompt_noise=0.25)
    scorer = train_ranking(train, TrainConfig(seed=0)).scorer
    scores = scorer.score_batch(reqs, 0)
    g = -np.asarray(scores, dtype=np.float64)
    order = np.argsort(ranking.bucket_lengths(lengths, 10), kind="stable")
    loss = ranking.list_mle_loss(g, order)
    grad = ranking.list_mle_gradient(g, order)
    for r, s in zip(reqs, scores):
        r.score = s
    dec = RankingPolicy(SchedulerConfig(max_batch=32, starvation_threshold=100, priority_quantum=50),
                        scorer.length_calibrated).schedule(reqs, 1 << 62)
    tau = ranking.kendall_tau_b(scores, lengths)
    out = {"generator": "make_cfg1_golden.py", "scores": [float(s) for s in scores],
           "lengths": [int(v) for v in lengths], "length_calibrated": bool(scorer.length_calibrated),
           "listmle_loss": float(loss), "listmle_grad": [float(v) for v in grad], "order": order.tolist(),
           "run": list(dec.run), "promoted": list(dec.promoted), "demoted": list(dec.demoted),
           "state": [[r.priority, r.starvation_count, r.quantum] for r in reqs],
           "tau": [tau.tau, tau.concordant, tau.discordant, tau.n_pairs]}
    OUT.write_text(json.dumps(out) + "\n")
    print("run", dec.run[:8], "tau", tau.tau, "loss", loss)


if __name__ == "__main__":
    main()

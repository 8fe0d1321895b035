"""B200-native hot path of the learning-to-rank request scheduler (arXiv 2408.15792).

Drop-in for the hot-path names of the reference package `ranksched`:

    from paper_2408_15792_b200 import kendall_tau_b, list_mle_loss, list_mle_gradient, \
        bucket_lengths, make_policy, SchedulerConfig, BatchDecision, OptRankerScorer

or, to make the reference's own engine / presets / CLI use the B200 kernels:

    import ranksched, paper_2408_15792_b200 as b200
    b200.install(ranksched)

All arithmetic runs in librsb200.so (sm_100a); there is no CPU fallback.
"""

from __future__ import annotations

import sys

from .ranking import (TauResult, bucket_lengths, kendall_tau_b, list_mle_batched, list_mle_gradient,  # noqa: F401
                      list_mle_loss, listmle_from_lengths, tau_counts_device)
from .schedulers import BatchDecision, DeviceQueue, RankingPolicy, SchedulerConfig, make_policy  # noqa: F401
from .workload import Request, RequestState  # noqa: F401

__version__ = "0.1.0"

_saved: dict = {}


def __getattr__(name):
    # the ranker / scorer pull in larger modules; import them lazily
    if name in ("OptRanker", "RankerConfig"):
        from . import ranker
        return getattr(ranker, name)
    if name in ("OptRankerScorer", "TrainConfig", "TrainResult", "save_scorer", "load_scorer", "scorer_from_dict",
                "train_ranking"):
        from . import predictors
        return getattr(predictors, name)
    raise AttributeError(name)


def install(ranksched) -> None:
    """Rebind the reference's hot-path entry points to the B200 implementations.

    * ranking.kendall_tau_b / list_mle_loss / list_mle_gradient everywhere the
      reference imported them (ranking, predictors, engine, the package namespace);
      kendall_tau_b returns the reference's own TauResult class;
    * engine.make_policy: "ranking" -> the device RankingPolicy (returning the
      reference's BatchDecision), every other policy name -> the reference's factory;
    * predictors.scorer_from_dict / load_scorer: kinds "opt-ranker" / "opt-classifier" ->
      OptRankerScorer / OptClassifierScorer, everything else -> the reference's if-chain.
    """
    import json

    from . import predictors as b_pred
    from . import ranking as b_rank
    from . import schedulers as b_sched

    mods = {name: sys.modules.get(f"{ranksched.__name__}.{name}") for name in
            ("ranking", "predictors", "engine", "presets", "cli")}
    mods["__init__"] = ranksched
    ref_ranking, ref_pred = mods["ranking"], mods["predictors"]
    ref_sched = sys.modules.get(f"{ranksched.__name__}.schedulers")
    RefTau = getattr(ref_ranking, "TauResult", b_rank.TauResult)
    RefDecision = getattr(ref_sched, "BatchDecision", b_sched.BatchDecision)

    def kendall_tau_b(x, y):
        r = b_rank.kendall_tau_b(x, y)
        return RefTau(r.tau, r.concordant, r.discordant, r.n_pairs)

    kendall_tau_b.__doc__ = b_rank.kendall_tau_b.__doc__

    class RankingPolicy(b_sched.RankingPolicy):
        decision_cls = RefDecision

    targets = {"kendall_tau_b": kendall_tau_b, "list_mle_loss": b_rank.list_mle_loss,
               "list_mle_gradient": b_rank.list_mle_gradient}
    ref_make_policy = mods["engine"].make_policy if mods["engine"] is not None else None
    ref_from_dict = ref_pred.scorer_from_dict if ref_pred is not None else None
    ref_load = ref_pred.load_scorer if ref_pred is not None else None
    ours = (b_pred.OptRankerScorer.kind, b_pred.OptClassifierScorer.kind)

    def make_policy(name, config, length_calibrated=True):
        if name.lower() == "ranking":
            return RankingPolicy(config, length_calibrated)
        return ref_make_policy(name, config, length_calibrated)

    def scorer_from_dict(obj):
        if obj.get("kind") in ours:
            return b_pred.scorer_from_dict(obj)
        return ref_from_dict(obj)

    def load_scorer(path):
        with open(path, "r", encoding="utf-8") as fh:
            kind = json.load(fh).get("kind")
        if kind in ours:
            return b_pred.load_scorer(path)  # same format / version checks, sidecar beside it
        return ref_load(path)

    rebinds = dict(targets, make_policy=make_policy, scorer_from_dict=scorer_from_dict, load_scorer=load_scorer)
    where = {"make_policy": ("engine", "presets", "cli"), "scorer_from_dict": ("predictors", "presets", "cli"),
             "load_scorer": ("predictors", "cli", "__init__")}
    for mname, mod in mods.items():
        if mod is None:
            continue
        for attr, new in rebinds.items():
            if attr in where and mname not in where[attr]:
                continue
            if hasattr(mod, attr):
                _saved.setdefault((id(mod), attr), (mod, getattr(mod, attr)))
                setattr(mod, attr, new)


def uninstall(ranksched=None) -> None:
    """Undo install()."""
    for (_, attr), (mod, old) in list(_saved.items()):
        setattr(mod, attr, old)
    _saved.clear()

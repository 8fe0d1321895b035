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
    * engine.make_policy: "ranking" -> the device RankingPolicy, every other policy
      name -> the reference's own factory;
    * predictors.scorer_from_dict / load_scorer: kinds "opt-ranker" / "opt-classifier" ->
      OptRankerScorer / OptClassifierScorer, everything else -> the reference's if-chain.
    """
    from . import predictors as b_pred
    from . import ranking as b_rank
    from . import schedulers as b_sched

    mods = {name: sys.modules.get(f"{ranksched.__name__}.{name}") for name in
            ("ranking", "predictors", "engine", "presets", "cli")}
    mods["__init__"] = ranksched
    targets = {"kendall_tau_b": b_rank.kendall_tau_b, "list_mle_loss": b_rank.list_mle_loss,
               "list_mle_gradient": b_rank.list_mle_gradient}
    ref_make_policy = mods["engine"].make_policy if mods["engine"] is not None else None
    ref_from_dict = mods["predictors"].scorer_from_dict if mods["predictors"] is not None else None

    def make_policy(name, config, length_calibrated=True):
        if name.lower() == "ranking":
            return b_sched.RankingPolicy(config, length_calibrated)
        return ref_make_policy(name, config, length_calibrated)

    def scorer_from_dict(obj):
        if obj.get("kind") in (b_pred.OptRankerScorer.kind, b_pred.OptClassifierScorer.kind):
            return b_pred.scorer_from_dict(obj)
        return ref_from_dict(obj)

    targets_mod = dict(targets)
    for mname, mod in mods.items():
        if mod is None:
            continue
        for attr, new in list(targets_mod.items()) + [("make_policy", make_policy),
                                                      ("scorer_from_dict", scorer_from_dict)]:
            if attr in ("make_policy",) and mname not in ("engine", "presets", "cli"):
                continue
            if attr == "scorer_from_dict" and mname not in ("predictors", "presets", "cli"):
                continue
            if hasattr(mod, attr):
                _saved.setdefault((id(mod), attr), (mod, getattr(mod, attr)))
                setattr(mod, attr, new)


def uninstall(ranksched=None) -> None:
    """Undo install()."""
    for (_, attr), (mod, old) in list(_saved.items()):
        setattr(mod, attr, old)
    _saved.clear()

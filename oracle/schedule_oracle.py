"""CPU restatement of the ranking policy — TEST INFRASTRUCTURE ONLY (checker).

Follows ranksched/schedulers.py:
  Policy._fill            :86-96   greedy, stop at max_batch, skip what does not fit
  Policy.schedule         :98-109  one sort (preemptive) or running-pinned + rest
  RankingPolicy.sort_key  :211-218 (unscored first, priority first, eff, arrival, id)
  RankingPolicy.schedule  :219-240 starvation count / quantum update, promote/demote
operating on plain dicts (or any objects with the Request attributes).
"""

from __future__ import annotations


def _running(r) -> bool:
    st = r.state
    return getattr(st, "value", st) == "running"


def effective_score(r, calibrated: bool) -> float:
    if r.score is None:
        return 0.0
    if calibrated:
        return r.score - r.generated_tokens
    return r.score


def sort_key(r, calibrated: bool):
    return (0 if r.score is None else 1, 0 if r.priority else 1, effective_score(r, calibrated),
            r.arrival_time, r.id)


def schedule(candidates, kv_budget, *, max_batch=256, preemption=True, threshold=100, quantum=50,
             calibrated=True):
    """One RankingPolicy.schedule step; mutates the candidates like the reference.
    Returns (run, promoted, demoted)."""
    key = lambda r: sort_key(r, calibrated)  # noqa: E731
    if preemption:
        ordered = sorted(candidates, key=key)
    else:
        ordered = sorted((r for r in candidates if _running(r)), key=key) + \
            sorted((r for r in candidates if not _running(r)), key=key)
    run = []
    used = 0
    for r in ordered:
        if len(run) >= max_batch:
            break
        need = r.prompt_tokens + r.generated_tokens + 1
        if used + need <= kv_budget:
            run.append(r)
            used += need
    run_ids = [r.id for r in run]
    sched = set(run_ids)
    promoted, demoted = [], []
    for r in candidates:
        if r.id in sched:
            r.starvation_count = 0
            if r.priority:
                r.quantum -= 1
        else:
            r.starvation_count += 1
    for r in candidates:
        if threshold > 0 and r.starvation_count >= threshold:
            r.priority = True
            r.quantum = quantum
            r.starvation_count = 0
            promoted.append(r.id)
        elif r.priority and r.quantum <= 0:
            r.priority = False
            demoted.append(r.id)
    return run_ids, promoted, demoted

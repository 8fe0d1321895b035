"""Host-side logic of the drop-in package (CPU)."""

import numpy as np
import pytest

from paper_2408_15792_b200 import schedulers, workload


def test_scheduler_config_validation_matches_reference():
    with pytest.raises(ValueError):
        schedulers.SchedulerConfig(max_batch=0)
    with pytest.raises(ValueError):
        schedulers.SchedulerConfig(starvation_threshold=-1)
    with pytest.raises(ValueError):
        schedulers.SchedulerConfig(priority_quantum=0)
    with pytest.raises(ValueError):
        schedulers.SchedulerConfig(mlfq_growth=0.5)
    schedulers.SchedulerConfig(starvation_threshold=0)


def test_make_policy():
    cfg = schedulers.SchedulerConfig()
    assert isinstance(schedulers.make_policy("RANKING", cfg), schedulers.RankingPolicy)
    with pytest.raises(ValueError):
        schedulers.make_policy("lifo", cfg)
    with pytest.raises(ValueError, match="baseline"):
        schedulers.make_policy("fcfs", cfg)


def test_sort_key_mirror():
    pol = schedulers.RankingPolicy(schedulers.SchedulerConfig(), length_calibrated=True)
    r = workload.Request(id=3, arrival_time=1.0, prompt_tokens=4, true_output_tokens=10)
    r.score, r.generated_tokens = 50.0, 45
    assert pol.sort_key(r) == (1, 1, 5.0, 1.0, 3)


def test_prompt_token_ids_deterministic_and_padded():
    ids, last = workload.prompt_token_ids("Hello world  how ARE you", 8)
    ids2, _ = workload.prompt_token_ids("hello WORLD how are you", 8)
    assert last == 4 and ids.dtype == np.int32 and ids.shape == (8,)
    np.testing.assert_array_equal(ids, ids2)  # lower-cased like featurize (workload.py:148)
    assert (ids[5:] == 1).all() and (ids[:5] >= 4).all() and (ids < 50272).all()
    ids, last = workload.prompt_token_ids("", 4)
    assert last == 0 and ids[0] == 2

"""Host-side pieces of the device engine (CPU): the cost model mirrors the reference's
(engine.py:42-93) and the latency-statistics arithmetic matches ranking.latency_stats."""

import math
import os
import sys

import pytest

from paper_2408_15792_b200 import engine



def test_cost_model_validation():
    with pytest.raises(ValueError):
        engine.CostModel(decode_ns=0)
    with pytest.raises(ValueError):
        engine.CostModel(prefill_ns_per_token=-1)
    with pytest.raises(ValueError):
        engine.CostModel(decode_table=(1, 0))
    assert engine.CostModel(decode_table=[3, 2]).decode_table == (3, 2)


def test_presets_and_stats_match_reference(ranksched):
    from ranksched import engine as ref_engine
    from ranksched.ranking import latency_stats
    for name, cm in ref_engine.COST_PRESETS.items():
        ours = engine.COST_PRESETS[name]
        assert (ours.decode_ns, ours.prefill_ns_per_token, ours.predictor_ns_per_request, ours.decode_table) == \
            (cm.decode_ns, cm.prefill_ns_per_token, cm.predictor_ns_per_request, cm.decode_table)
    lat, ptl, mw = [3.0, 1.5, 2.25, 9.0, 0.5], [0.3, 0.1, 0.2, 0.9, 0.05], [1.0, 0.5, 0.25, 4.0, 0.125]
    ref = latency_stats(lat, ptl, mw, makespan=12.5)
    ours = engine._latency_stats(lat, ptl, mw, 12.5)
    assert ours["mean_latency"] == ref.mean_latency and ours["p90_latency"] == ref.p90_latency
    assert ours["mean_max_waiting_time"] == ref.mean_max_waiting_time
    assert ours["p90_per_token_latency"] == ref.p90_per_token_latency
    assert math.isclose(ours["throughput"], ref.throughput)
    empty = engine._latency_stats([], [], [], 3.0)
    assert empty["makespan"] == 3.0 and empty["throughput"] == 0.0

"""§8f #2 trace formats and generators vs the staged reference (CPU): the same (spec,
seed) yields the identical trace (fingerprint, metadata, per-request fields), JSONL
round trips, and the reference's validation errors."""

import json

import numpy as np
import pytest

from paper_2408_15792_b200 import workload as w


def _same(a, b):
    assert a.fingerprint() == b.fingerprint()
    assert a.metadata == b.metadata
    assert [(r.id, r.arrival_time, r.prompt_tokens, r.true_output_tokens, r.prompt) for r in a] == \
        [(r.id, r.arrival_time, r.prompt_tokens, r.true_output_tokens, r.prompt) for r in b]


@pytest.mark.parametrize("spec", [
    "poisson:rate=40,n=3000,dist=sharegpt,seed=7,pnoise=0.25",
    "poisson:rate=2,n=500,dist=lognormal(5.0,1.0),seed=7",
    "burst:n=800,dist=lmsys,seed=3,pnoise=0.5",
    "burst:n=300,dist=uniform(1,400),seed=11",
    "poisson:rate=5.5,n=200,dist=geometric(0.01),seed=1,pnoise=0.1",
])
def test_generators_match_reference(ranksched, spec):
    _same(w.parse_generator_spec(spec), ranksched.workload.parse_generator_spec(spec))


def test_fixed_resample_features_match_reference(ranksched):
    rw = ranksched.workload
    _same(w.fixed_burst([5, 1, 9, 3]), rw.fixed_burst([5, 1, 9, 3]))
    t = w.generate_burst(400, w.LengthDist.parse("sharegpt"), seed=2, prompt_noise=0.3)
    rt = rw.generate_burst(400, rw.LengthDist.parse("sharegpt"), seed=2, prompt_noise=0.3)
    _same(w.resample_lengths(t, 9, 0.4), rw.resample_lengths(rt, 9, 0.4))
    for r, q in zip(t, rt):
        assert np.array_equal(r.features, q.features)
    for p in ["", "What?  EXPLAIN list-code", "  über  naïve \t x\ny ", "a" * 5000, "code " * 3000]:
        assert np.array_equal(w.featurize(p), rw.featurize(p))


def test_jsonl_round_trip_and_reference_loader(ranksched, tmp_path):
    t = w.parse_generator_spec("poisson:rate=10,n=200,dist=sharegpt,seed=4,pnoise=0.2")
    p = tmp_path / "t.jsonl"
    w.save_trace(t, str(p))
    back = w.load_trace(str(p))
    ref = ranksched.workload.load_trace(str(p))
    _same(back, ref)
    assert [r.prompt for r in back] == [r.prompt for r in t]
    # the reference's writer produces the same bytes
    p2 = tmp_path / "r.jsonl"
    ranksched.workload.save_trace(ref, str(p2))
    assert p.read_bytes() == p2.read_bytes()
    # unsorted arrivals and missing arrival_time are accepted and ordered like the reference
    p3 = tmp_path / "u.jsonl"
    p3.write_text("\n".join(json.dumps(o) for o in [
        {"prompt": "b b", "output_tokens_length": 3, "arrival_time": 2.0},
        {"prompt": "a", "output_tokens_length": 1},
        {"prompt": "c c c", "output_tokens_length": 7, "arrival_time": 1.0}]) + "\n\n")
    _same(w.load_trace(str(p3)), ranksched.workload.load_trace(str(p3)))


@pytest.mark.parametrize("body,msg", [
    ("{bad", "malformed JSON"), ('{"output_tokens_length": 3}', "missing 'prompt'"),
    ('{"prompt": "x"}', "missing 'output_tokens_length'"),
    ('{"prompt": "x", "output_tokens_length": 0}', "positive int"),
    ('{"prompt": "x", "output_tokens_length": 2.0}', "positive int"),
    ('{"prompt": "x", "output_tokens_length": 2, "arrival_time": -1}', "negative arrival_time")])
def test_load_trace_errors(tmp_path, body, msg):
    p = tmp_path / "bad.jsonl"
    p.write_text(body + "\n")
    with pytest.raises(ValueError, match=msg):
        w.load_trace(str(p))


@pytest.mark.parametrize("spec", ["poisson", "poisson:rate=1,n=5", "nope:n=3,dist=sharegpt",
                                  "poisson:n=3,dist=sharegpt", "burst:n=3,dist=wat(1)", "burst:n=3,dist=uniform(5,1)",
                                  "burst:n=0,dist=sharegpt", "poisson:rate=0,n=3,dist=sharegpt", "burst:n=3,dist"])
def test_generator_spec_errors(spec):
    with pytest.raises(ValueError):
        w.parse_generator_spec(spec)

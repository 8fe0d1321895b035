"""The one-launch engine loop (rs_engine_run's device path, csrc/rankstep.cu
engine_loop_kernel) against the per-kernel host loop (RS_ENGINE_LOOP=host) on the
configurations the loop handles differently: length-calibrated keys, non-preemptive
pinning, stop-after-finished and time-limit exits, the largest batch the fused select
takes (512), no predictor charge, a KV budget (which keeps the host loop), a burst
admitted in one step, and a batch of one. Same
per-request rows, metrics and step counts. The host loop's decisions are checked step for
step against the reference's engine.run in test_gpu_engine.py."""

import json
import os
import pathlib
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HELPER = pathlib.Path(__file__).resolve().parent / "engine_loop_case.py"
CASES = ["calibrated", "non_preemptive", "stop_after", "time_limit", "max_batch_512", "no_predictor_charge",
         "kv_budget", "burst", "max_batch_1"]


def _run(name, host):
    env = dict(os.environ)
    env.pop("RS_ENGINE_LOOP", None)
    if host:
        env["RS_ENGINE_LOOP"] = "host"
    p = subprocess.run([sys.executable, str(HELPER), name], env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("name", CASES)
def test_device_loop_equals_host_loop(name):
    dev, host = _run(name, False), _run(name, True)
    assert dev["steps"] == host["steps"]
    assert dev["metrics"] == host["metrics"]
    assert dev["rows"] == host["rows"]
    assert dev["steps"] > 0

"""The N > 1 bench path (score shards, all-gather to rank 0, rank-step, max-over-ranks
timing) run as two ranks on the test box's one GPU over gloo (NCCL refuses two ranks per
device; the driver's multi-GPU runs use NCCL on separate GPUs)."""

import json
import os
import pathlib
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent


@pytest.mark.gpu
def test_bench_two_ranks_gloo():
    env = dict(os.environ, RSB200_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29541", str(ROOT / "bench.py"), "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--batch", "256", "--seq", "128", "--no-extras"]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-3000:]  # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["config"]["global_batch"] == 512
    assert line["config"]["parallelism"] == "dp2" and line["value"] > 0 and line["gpu_launches"] > 0


@pytest.mark.gpu
def test_bench_self_launches_ranks():
    """`python bench.py --gpus 2` with no launcher in the environment starts its own two
    ranks (torch.distributed.run on 127.0.0.1) and reports n_gpus == 2."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["RSB200_BENCH_BACKEND"] = "gloo"
    cmd = [sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--batch", "128", "--seq", "128", "--no-extras"]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-3000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["config"]["global_batch"] == 256 and line["config"]["parallelism"] == "dp2"

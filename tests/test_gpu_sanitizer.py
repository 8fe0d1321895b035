"""compute-sanitizer over small shapes of every kernel (tools/sanitize_small.py): memcheck
(out-of-bounds / misaligned device accesses, leaks), racecheck (shared-memory hazards),
synccheck (illegal barrier use) and initcheck (reads of uninitialised device memory).
The hand-rolled mbarrier / TMEM / TMA protocols of the tcgen05 kernels are the reason
this exists."""

import os
import pathlib
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = pathlib.Path(__file__).resolve().parents[1]


def _sanitizer():
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(exe):
        pytest.skip("compute-sanitizer not installed")
    return exe


@pytest.mark.parametrize("tool,part", [("memcheck", "all"), ("synccheck", "all"), ("racecheck", "sort"),
                                       ("racecheck", "engine"), ("racecheck", "ranker"), ("initcheck", "sort")])
def test_compute_sanitizer_clean(tool, part):
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "99", "--print-limit", "20"]
    cmd += [sys.executable, str(ROOT / "tools" / "sanitize_small.py"), part]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    text = out.stdout + out.stderr
    assert "sanitize-small ok" in text, text[-4000:]
    assert out.returncode == 0 and "ERROR SUMMARY: 0 errors" in text, text[-4000:]

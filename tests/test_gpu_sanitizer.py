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
    # some GPU pools replace the tool by a stub that refuses every run ("closed on this
    # pool"); probe it once without launching anything under it
    probe = subprocess.run([exe, "--version"], capture_output=True, text=True, timeout=60)
    text = probe.stdout + probe.stderr
    if probe.returncode != 0 or "closed" in text:
        pytest.skip("compute-sanitizer unavailable on this box: " + text.strip()[:200])
    return exe


# racecheck / synccheck do not model the tcgen05 machinery: racecheck reports the
# warp-collective tcgen05.alloc (the tensor core writing the TMEM base address into shared
# memory) as a race with the alloc instruction itself, at an unattributable kernel offset,
# and synccheck reports the tcgen05 kernels' first mbarrier parity waits as "missing init"
# although the barriers are initialised, fenced (fence.mbarrier_init) and published by
# __syncthreads before any wait (attention.cu:172-204; plain-mbarrier probes in
# tools/probes/ are clean under the same tool). Those kernels (the GEMMs and the
# attention forward / backward) are covered by memcheck here and by the numerics tests;
# the two tools check every other kernel.
_TCGEN05 = ["--kernel-name-exclude", "regex=gemm_bf16|attention_fwd|attention_bwd"]


@pytest.mark.parametrize("tool,part", [("memcheck", "all"), ("synccheck", "all"), ("racecheck", "sort"),
                                       ("racecheck", "engine"), ("racecheck", "ranker"), ("initcheck", "sort")])
def test_compute_sanitizer_clean(tool, part):
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "99", "--print-limit", "20"]
    if tool in ("racecheck", "synccheck"):
        cmd += _TCGEN05
    cmd += [sys.executable, str(ROOT / "tools" / "sanitize_small.py"), part]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    text = out.stdout + out.stderr
    assert "sanitize-small ok" in text, text[-4000:]
    summary = "RACECHECK SUMMARY: 0 hazards" if tool == "racecheck" else "ERROR SUMMARY: 0 errors"
    assert out.returncode == 0 and summary in text, text[-4000:]

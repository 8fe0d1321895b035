"""Stage the reference package `ranksched` under oracle/_ref/ — TEST INFRASTRUCTURE ONLY.

The reference (/root/reference/pkg, pure Python + numpy) is the oracle for every integer
row of the hot path and the CPU baseline the bench times beside the GPU. /root/reference
exists only in the build container, so build() stages an unmodified copy of its package
directory here (git-ignored, not gpurun-ignored: it travels to the GPU box with the
snapshot, like a built .so). Nothing in paper_2408_15792_b200 imports it; tests/,
smoke() and bench.py's cpu_baseline / --impl reference arm put oracle/_ref on sys.path.

    python oracle/install_ref.py [--src /root/reference/pkg/src/ranksched]
"""

from __future__ import annotations

import argparse
import hashlib
import json
import pathlib
import shutil
import sys

HERE = pathlib.Path(__file__).resolve().parent
DEST = HERE / "_ref"
SRC = pathlib.Path("/root/reference/pkg/src/ranksched")


def tree_sha(root: pathlib.Path) -> str:
    h = hashlib.sha256()
    for p in sorted(root.rglob("*.py")):
        h.update(p.relative_to(root).as_posix().encode())
        h.update(p.read_bytes())
    return h.hexdigest()


def install(src: pathlib.Path = SRC) -> bool:
    if not src.is_dir():
        return False
    dst = DEST / "ranksched"
    want = tree_sha(src)
    stamp = DEST / "STAMP.json"
    if dst.is_dir() and stamp.exists() and json.loads(stamp.read_text()).get("sha256") == want:
        return True
    if dst.exists():
        shutil.rmtree(dst)
    DEST.mkdir(parents=True, exist_ok=True)
    shutil.copytree(src, dst, ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
    stamp.write_text(json.dumps({"source": str(src), "sha256": want}) + "\n")
    return True


def available() -> bool:
    return (DEST / "ranksched" / "__init__.py").exists()


def import_ranksched():
    """Import the staged reference (raises ImportError when it was not staged)."""
    if not available():
        raise ImportError("oracle/_ref/ranksched is not staged (run oracle/install_ref.py where "
                          "/root/reference exists)")
    p = str(DEST)
    if p not in sys.path:
        sys.path.insert(0, p)
    import ranksched  # noqa: F401
    import ranksched.engine  # noqa: F401
    import ranksched.predictors  # noqa: F401
    import ranksched.ranking  # noqa: F401
    import ranksched.schedulers  # noqa: F401
    import ranksched.workload  # noqa: F401
    return sys.modules["ranksched"]


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--src", default=str(SRC))
    ok = install(pathlib.Path(ap.parse_args().src))
    print("staged" if ok else "reference source absent; nothing staged")

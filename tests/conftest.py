import pathlib
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
for p in (str(ROOT), str(ROOT / "tests" / "golden")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built librsb200.so")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    import json
    d = ROOT / "tests" / "golden"
    return {p.stem: json.loads(p.read_text()) for p in d.glob("*.json")}


@pytest.fixture(scope="session")
def ranksched():
    """The reference package, staged under oracle/_ref by build() (travels to the GPU box);
    skips when it was never staged."""
    from oracle import install_ref
    try:
        return install_ref.import_ranksched()
    except ImportError as e:
        pytest.skip(str(e))

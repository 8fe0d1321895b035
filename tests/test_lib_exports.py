"""The C-ABI library loads and exports every symbol include/rsb200.h declares (CPU)."""

import ctypes
import re

from paper_2408_15792_b200 import _lib
from conftest import ROOT


def declared_symbols():
    text = (ROOT / "include" / "rsb200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rs_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 15
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # the ctypes signature table covers exactly the declared ABI
    assert sorted(_lib.SIGNATURES) == syms


def test_host_only_entry_points():
    lib = _lib.load()
    assert lib.rs_version() == 1
    assert lib.rs_tau_workspace_size(1 << 20, _lib.RS_F32, _lib.RS_I32) > 8 << 20
    assert lib.rs_rank_step_workspace_size(1000) > 0
    assert lib.rs_arrival_rank_workspace_size(1000) > 0
    # bad argument -> ValueError with the C message, no device touched
    import pytest
    with pytest.raises(ValueError, match="dtype"):
        _lib.check(lib.rs_tau_counts(None, 9, None, 0, 10, None, None, 0, None))

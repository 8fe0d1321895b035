"""ctypes wrapper of oracle/tau_pairs.c — TEST INFRASTRUCTURE ONLY (checker / CPU baseline)."""

from __future__ import annotations

import ctypes
import os
import pathlib
import subprocess

import numpy as np

_HERE = pathlib.Path(__file__).resolve().parent
_SO = _HERE / "_build" / "libtau_oracle.so"
_lib = None


def build() -> pathlib.Path:
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _SO


def _load():
    global _lib
    if _lib is None:
        if not _SO.exists():
            build()
        lib = ctypes.CDLL(str(_SO))
        lib.tau_pairs_f64.restype = ctypes.c_int
        lib.tau_pairs_f64.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                      ctypes.c_int]
        _lib = lib
    return _lib


def tau_counts(x, y, threads: int | None = None):
    """(C, D, n1, n2, n3) by exhaustive pair enumeration in C (ranking.py:45-57)."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    y = np.ascontiguousarray(np.asarray(y, dtype=np.float64))
    if x.shape != y.shape or x.ndim != 1:
        raise ValueError("kendall_tau_b expects two equal-length 1-d arrays")
    out = np.zeros(5, dtype=np.int64)
    t = threads or os.cpu_count() or 1
    rc = _load().tau_pairs_f64(x.ctypes.data, y.ctypes.data, len(x), out.ctypes.data, t)
    if rc != 0:
        raise RuntimeError("tau_pairs_f64 failed")
    return tuple(int(v) for v in out)

"""ctypes binding of librsb200.so (the C ABI declared in include/rsb200.h).

There is no fallback: if the shared library is missing or the device is not an
sm_100 part, every entry point raises. Device memory and streams come from torch
(plumbing only); every compute call goes through the C ABI.
"""

from __future__ import annotations

import ctypes
import os
import pathlib
import threading

import torch

_LIB_PATH = pathlib.Path(
    os.environ.get("RSB200_LIB", str(pathlib.Path(__file__).with_name("librsb200.so"))))

RS_OK = 0
RS_ERR_INVALID = -1
RS_ERR_CUDA = -2
RS_ERR_NAN = -3
RS_ERR_NOT_PERMUTATION = -4
RS_ERR_WORKSPACE = -5
RS_ERR_UNSUPPORTED = -6

RS_F32, RS_F64, RS_I32, RS_I64, RS_BF16 = 0, 1, 2, 3, 4

RS_FLAG_SCORED, RS_FLAG_PRIORITY, RS_FLAG_RUNNING = 1, 2, 4

c_i32, c_i64, c_sz, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t, ctypes.c_void_p


class RankerConfig(ctypes.Structure):
    _fields_ = [("vocab", c_i32), ("max_pos", c_i32), ("d_model", c_i32), ("n_layers", c_i32),
                ("n_heads", c_i32), ("d_ffn", c_i32), ("activation", c_i32)]


class QueueSoA(ctypes.Structure):
    _fields_ = [("n", c_i64), ("score_dtype", c_i32), ("score", c_vp), ("prompt_tokens", c_vp),
                ("generated_tokens", c_vp), ("arrival_rank", c_vp), ("id", c_vp), ("flags", c_vp),
                ("starvation", c_vp), ("quantum", c_vp)]


class EngineQueue(ctypes.Structure):
    _fields_ = [("n", c_i64), ("score_dtype", c_i32), ("score", c_vp), ("prompt_tokens", c_vp),
                ("generated_tokens", c_vp), ("arrival_rank", c_vp), ("id", c_vp), ("flags", c_vp),
                ("starvation", c_vp), ("quantum", c_vp)]


class EngineTrace(ctypes.Structure):
    _fields_ = [("score", c_vp), ("prompt_tokens", c_vp), ("true_output", c_vp), ("arrival_rank", c_vp),
                ("arrival_ns", c_vp), ("row_of", c_vp), ("run_stamp", c_vp), ("first_token_ns", c_vp),
                ("last_event_ns", c_vp), ("max_gap_ns", c_vp), ("finish_ns", c_vp), ("n_preempted", c_vp)]


class EngineCost(ctypes.Structure):
    _fields_ = [("decode_ns", c_i64), ("prefill_ns_per_token", c_i64), ("decode_table", c_vp),
                ("decode_table_len", c_i32)]


class EngineLoop(ctypes.Structure):
    _fields_ = [("n_requests", c_i64), ("arrival_ns", c_vp), ("fits", c_vp), ("adm_host", c_vp), ("adm_dev", c_vp),
                ("dropped_host", c_vp), ("stat_dev", c_vp), ("stat_host", c_vp), ("run_dev", c_vp),
                ("prom_dev", c_vp), ("dem_dev", c_vp), ("pre_dev", c_vp), ("fin_dev", c_vp), ("scratch_dev", c_vp),
                ("prev_run_dev", c_vp), ("prev_n_dev", c_vp), ("ws", c_vp), ("ws_bytes", c_sz), ("max_batch", c_i32), ("starvation_threshold", c_i32),
                ("priority_quantum", c_i32), ("length_calibrated", c_i32), ("preemptive", c_i32),
                ("kv_budget", c_i64), ("predictor_ns_per_request", c_i64), ("limit_ns", c_i64),
                ("stop_after_finished", c_i64)]


class EngineLoopOut(ctypes.Structure):
    _fields_ = [("now_ns", c_i64), ("steps", c_i64), ("n_finished", c_i64), ("next_arrival", c_i64),
                ("n_dropped", c_i64), ("total_prefill_ns", c_i64), ("total_decode_ns", c_i64),
                ("total_predictor_ns", c_i64), ("final_set", c_i32)]


# name -> (restype, argtypes); the list mirrors include/rsb200.h exactly and
# tests/test_lib_exports.py checks every declared symbol is exported.
SIGNATURES = {
    "rs_last_error": (ctypes.c_char_p, []),
    "rs_version": (ctypes.c_int, []),
    "rs_device_init": (ctypes.c_int, [ctypes.c_int, c_vp, c_vp, c_vp]),
    "rs_tau_workspace_size": (c_sz, [c_i64, ctypes.c_int, ctypes.c_int]),
    "rs_tau_counts": (ctypes.c_int, [c_vp, ctypes.c_int, c_vp, ctypes.c_int, c_i64, c_vp, c_vp, c_sz, c_vp]),
    "rs_tau_counts_fast": (ctypes.c_int, [c_vp, ctypes.c_int, c_vp, ctypes.c_int, c_i64, c_vp, c_vp, c_sz, c_vp]),
    "rs_listmle_order": (ctypes.c_int, [c_vp, ctypes.c_int, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "rs_listmle_lengths": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp]),
    "rs_arrival_rank_workspace_size": (c_sz, [c_i64]),
    "rs_arrival_rank": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_sz, c_vp]),
    "rs_engine_admit": (ctypes.c_int, [ctypes.POINTER(EngineQueue), ctypes.POINTER(EngineTrace), c_vp, c_i32, c_i64,
                                       c_vp]),
    "rs_engine_execute": (ctypes.c_int, [ctypes.POINTER(EngineQueue), ctypes.POINTER(EngineTrace),
                                         ctypes.POINTER(EngineCost), c_vp, c_vp, c_i32, c_i64, c_vp, c_vp, c_vp,
                                         c_vp]),
    "rs_engine_execute_ex": (ctypes.c_int, [ctypes.POINTER(EngineQueue), ctypes.POINTER(EngineQueue),
                                            ctypes.POINTER(EngineTrace), ctypes.POINTER(EngineCost), c_vp, c_vp, c_i32,
                                            c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "rs_tokenize": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, ctypes.c_uint32, c_vp, c_vp, c_vp, c_vp]),
    "rs_engine_run": (ctypes.c_int, [ctypes.POINTER(EngineQueue), ctypes.POINTER(QueueSoA), ctypes.POINTER(EngineTrace),
                                     ctypes.POINTER(EngineCost), ctypes.POINTER(EngineLoop),
                                     ctypes.POINTER(EngineLoopOut), c_vp]),
    "rs_rank_step_workspace_size": (c_sz, [c_i64]),
    "rs_rank_step": (ctypes.c_int, [ctypes.POINTER(QueueSoA), c_i32, c_i64, c_i32, c_i32, c_i32, c_i32,
                                    c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "rs_ranker_layout": (c_i64, [ctypes.POINTER(RankerConfig), c_vp]),
    "rs_ranker_workspace_size": (c_sz, [ctypes.POINTER(RankerConfig), c_i32, c_i32]),
    "rs_ranker_forward": (ctypes.c_int, [ctypes.POINTER(RankerConfig), c_vp, c_vp, c_vp, c_i32, c_i32, c_vp,
                                         c_vp, c_vp, c_sz, c_vp]),
    "rs_ranker_forward_ex": (ctypes.c_int, [ctypes.POINTER(RankerConfig), c_vp, c_vp, c_vp, c_i32, c_i32, c_vp,
                                            c_vp, c_vp, c_vp, c_sz, c_vp]),
    "rs_cls_logits": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_vp, c_vp]),
    "rs_cls_ce": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "rs_ranker_grad_cls_workspace_size": (c_sz, [ctypes.POINTER(RankerConfig), c_i32, c_i32, c_i32]),
    "rs_ranker_grad_cls": (ctypes.c_int, [ctypes.POINTER(RankerConfig), c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_i32,
                                          c_i32, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_sz, c_vp]),
    "rs_gemm_bf16": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_vp]),
    "rs_attention_fwd": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i32, c_i32, c_vp]),
    "rs_attention_fwd_f16v": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i32, c_i32, c_vp]),
    "rs_launch_count": (ctypes.c_uint64, []),
    "rs_ranker_grad_workspace_size": (c_sz, [ctypes.POINTER(RankerConfig), c_i32, c_i32, c_i32]),
    "rs_ranker_grad": (ctypes.c_int, [ctypes.POINTER(RankerConfig), c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32,
                                      c_i32, c_i32, c_vp, c_vp, c_sz, c_vp]),
    "rs_adam_step": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, ctypes.c_float, ctypes.c_float,
                                    ctypes.c_float, ctypes.c_float, c_i64, ctypes.c_float, c_vp]),
    "rs_attention_bwd": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_vp]),
    "rs_attention_fwd_lse": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_vp]),
    "rs_attention_bwd_lse": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_vp]),
    "rs_attention_bwd_long_workspace_size": (c_sz, [c_i32, c_i32, c_i32]),
    "rs_attention_bwd_long": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_vp, c_sz, c_vp]),
    "rs_attention_bwd_long_lse": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_vp, c_sz,
                                                 c_vp]),
    "rs_linear_n_params": (c_i64, [c_i32, c_i32]),
    "rs_standardizer_fit": (ctypes.c_int, [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp]),
    "rs_standardize": (ctypes.c_int, [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "rs_linear_forward": (ctypes.c_int, [c_vp, c_i64, c_i32, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp]),
    "rs_linear_train_step": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp,
                                            ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                            c_i64, c_vp, c_vp, c_vp]),
    "rs_gemm_bf16_ex": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32,
                                       c_vp]),
}

_lock = threading.Lock()
_lib = None
_inited_devices: dict[int, int] = {}


def lib_path() -> pathlib.Path:
    return _LIB_PATH


def load() -> ctypes.CDLL:
    """Load librsb200.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not _LIB_PATH.exists():
                raise RuntimeError(
                    f"{_LIB_PATH} not found: build it with `make -C paper_2408_15792_b200/csrc` "
                    "or __graft_entry__.build(); the B200 path has no CPU fallback")
            lib = ctypes.CDLL(str(_LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name, None)
                if fn is None:  # surfaces as AttributeError at the call site
                    continue
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def last_error() -> str:
    msg = load().rs_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = "") -> None:
    if status == RS_OK:
        return
    msg = last_error() or what
    if status in (RS_ERR_INVALID, RS_ERR_NAN, RS_ERR_NOT_PERMUTATION, RS_ERR_WORKSPACE):
        raise ValueError(msg)
    raise RuntimeError(f"rsb200 error {status}: {msg}")


def device(index: int | None = None) -> torch.device:
    """The CUDA device the kernels run on (initialised once per process)."""
    if not torch.cuda.is_available():
        raise RuntimeError("rsb200 needs a CUDA device (B200, sm_100a); none is visible")
    idx = torch.cuda.current_device() if index is None else index
    if idx not in _inited_devices:
        sm, ma, mi = c_i32(), c_i32(), c_i32()
        check(load().rs_device_init(idx, ctypes.byref(sm), ctypes.byref(ma), ctypes.byref(mi)),
              "rs_device_init")
        _inited_devices[idx] = sm.value
    return torch.device("cuda", idx)


def sm_count(index: int | None = None) -> int:
    d = device(index)
    return _inited_devices[d.index]


def stream_handle(dev: torch.device | None = None) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


class Workspace:
    """Grow-only per-device scratch buffer handed to the C ABI."""

    def __init__(self):
        self._bufs: dict[int, torch.Tensor] = {}

    def get(self, nbytes: int, dev: torch.device) -> tuple[int, int]:
        buf = self._bufs.get(dev.index)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(int(nbytes), 1 << 20), dtype=torch.uint8, device=dev)
            self._bufs[dev.index] = buf
        return buf.data_ptr(), buf.numel()


workspace = Workspace()

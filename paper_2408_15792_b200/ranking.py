"""Rank correlation and listwise loss on the B200 (drop-in for ranksched.ranking).

Same names, signatures, return types and error behaviour as the reference module
(ranksched/ranking.py); the arithmetic runs in librsb200 kernels:

* kendall_tau_b      -> rs_tau_counts (exact int64 C, D, n1, n2, n3), tau finished
                         here with the reference's own expression (ranking.py:58-63)
* list_mle_loss /    -> rs_listmle_order (warp-segmented log-sum-exp scans, float64
  list_mle_gradient     for float64 input exactly like ranking.py:86-120)
* listmle_from_lengths / list_mle_batched -> the batched device entry points used by
  the trainer (predictors.py:379-384 fused: bucketing + stable order + loss + grad)

Inputs may be numpy arrays / lists (copied host->device) or CUDA tensors (used in
place). bucket_lengths is integer floor division (ranking.py:123-132); on CUDA tensors
it runs on the device, and inside training it is fused into rs_listmle_lengths.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


@dataclass(frozen=True)
class TauResult:
    tau: float
    concordant: int
    discordant: int
    n_pairs: int


_TORCH_DT = {torch.float32: _lib.RS_F32, torch.float64: _lib.RS_F64,
             torch.int32: _lib.RS_I32, torch.int64: _lib.RS_I64}


def _as_device_1d(v, dev) -> torch.Tensor:
    """Numeric 1-d input -> CUDA tensor in one of the four kernel dtypes."""
    if isinstance(v, torch.Tensor):
        t = v.detach()
        if t.dtype not in _TORCH_DT:
            if t.dtype.is_floating_point:
                t = t.to(torch.float64)
            else:
                t = t.to(torch.int64)
        return t.to(dev).contiguous()
    a = np.asarray(v)
    if a.dtype == np.float32 or a.dtype == np.float64 or a.dtype == np.int32 or a.dtype == np.int64:
        pass
    elif a.dtype.kind in "biu" and a.dtype != np.uint64:
        a = a.astype(np.int64)
    else:
        # same float64 view the reference takes (np.asarray(x, dtype=np.float64))
        a = np.asarray(v, dtype=np.float64)
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev, non_blocking=False)


def tau_counts_device(x: torch.Tensor, y: torch.Tensor, out: torch.Tensor | None = None,
                      fast_only: bool = False) -> torch.Tensor:
    """Exact pair counts int64[6] = (C, D, n1, n2, n3, status) for CUDA tensors; status 1 =
    NaN seen. rs_tau_counts runs the bucket fast path (y spanning < 4096 values) and reads
    its status once, falling back to the general path when needed; with `fast_only` the
    call never synchronises and status 2 means "needs the general path" (call again
    without fast_only)."""
    dev = x.device
    n = x.numel()
    lib = _lib.load()
    if out is None:
        out = torch.empty(6, dtype=torch.int64, device=dev)
    xd, yd = _TORCH_DT[x.dtype], _TORCH_DT[y.dtype]
    ws_need = lib.rs_tau_workspace_size(n, xd, yd)
    ws, ws_n = _lib.workspace.get(ws_need, dev)
    fn, name = (lib.rs_tau_counts_fast, "rs_tau_counts_fast") if fast_only else (lib.rs_tau_counts, "rs_tau_counts")
    _lib.check(fn(x.data_ptr(), xd, y.data_ptr(), yd, n, out.data_ptr(), ws, ws_n, _lib.stream_handle(dev)), name)
    return out


class TauPlan:
    """rs_tau_counts_fast for fixed device inputs, captured once as a CUDA graph.

    At ~1M rows the exact count is launch-bound (~13 small kernels); a graph replays them
    with one launch. x, y and out must keep their storage for the plan's lifetime (the
    graph holds their addresses); the plan owns its workspace. `plan()` replays without
    synchronising (out[5] == 2 if these inputs need the general path); `plan.counts()`
    replays, checks, and falls back to the eager general path when needed.
    """

    def __init__(self, x: torch.Tensor, y: torch.Tensor, out: torch.Tensor | None = None):
        if x.numel() != y.numel() or not x.is_cuda or not y.is_cuda:
            raise ValueError("TauPlan expects two equal-length CUDA tensors")
        self.x, self.y = x, y
        self.dev = x.device
        self.out = out if out is not None else torch.empty(6, dtype=torch.int64, device=self.dev)
        lib = _lib.load()
        self._xd, self._yd = _TORCH_DT[x.dtype], _TORCH_DT[y.dtype]
        self._ws = torch.empty(max(lib.rs_tau_workspace_size(x.numel(), self._xd, self._yd), 1), dtype=torch.uint8,
                               device=self.dev)
        self._call()  # eager once (one-time kernel attributes), then capture
        torch.cuda.synchronize(self.dev)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._call()

    def _call(self):
        lib = _lib.load()
        _lib.check(lib.rs_tau_counts_fast(self.x.data_ptr(), self._xd, self.y.data_ptr(), self._yd, self.x.numel(),
                                          self.out.data_ptr(), self._ws.data_ptr(), self._ws.numel(),
                                          _lib.stream_handle(self.dev)), "rs_tau_counts_fast")

    def __call__(self) -> torch.Tensor:
        self.graph.replay()
        return self.out

    def counts(self) -> torch.Tensor:
        self.graph.replay()
        if int(self.out[5]) == 2:
            lib = _lib.load()
            _lib.check(lib.rs_tau_counts(self.x.data_ptr(), self._xd, self.y.data_ptr(), self._yd, self.x.numel(),
                                         self.out.data_ptr(), self._ws.data_ptr(), self._ws.numel(),
                                         _lib.stream_handle(self.dev)), "rs_tau_counts")
        return self.out


def tau_from_counts(counts, n: int) -> TauResult:
    """Finish tau exactly as the reference does (ranking.py:58-63), on Python ints."""
    c, d, n1, n2, _n3, nan = (int(v) for v in counts)
    if nan:
        raise ValueError("tau counts of NaN input: use kendall_tau_b, which handles NaN like the reference")
    return _finish(c, d, n1, n2, n)


def _finish(c: int, d: int, n1: int, n2: int, n: int) -> TauResult:
    n0 = n * (n - 1) // 2
    denom = math.sqrt((n0 - n1) * (n0 - n2))
    if denom == 0.0:
        return TauResult(0.0, c, d, n0)
    return TauResult((c - d) / denom, c, d, n0)


def kendall_tau_b(x, y) -> TauResult:
    """Kendall rank correlation, tau-b normalisation (drop-in for ranking.py:24-63)."""
    xs = x.shape if isinstance(x, torch.Tensor) else np.shape(np.asarray(x, dtype=np.float64))
    ys = y.shape if isinstance(y, torch.Tensor) else np.shape(np.asarray(y, dtype=np.float64))
    if tuple(xs) != tuple(ys) or len(xs) != 1:
        raise ValueError("kendall_tau_b expects two equal-length 1-d arrays")
    n = int(xs[0])
    if n * (n - 1) // 2 == 0:
        return TauResult(0.0, 0, 0, 0)
    dev = _lib.device()
    xt = _as_device_1d(x, dev)
    yt = _as_device_1d(y, dev)
    counts = tau_counts_device(xt, yt).cpu().tolist()
    if counts[5] == 1:
        return _tau_with_nan(xt, yt, n)
    return tau_from_counts(counts, n)


def _pairs(k: int) -> int:
    return k * (k - 1) // 2


def _tau_with_nan(xt: torch.Tensor, yt: torch.Tensor, n: int) -> TauResult:
    """NaN input, as the reference treats it (ranking.py:45-57): a pair with a NaN in x or y
    has sign(NaN) = NaN and counts as neither concordant nor discordant, and np.unique
    (equal_nan) puts all NaNs of a column in one tie group. So C, D are the counts over
    the rows NaN-free in both columns, and n1 (n2) = ties among x's (y's) non-NaN values +
    the pairs among its NaNs; every count still comes from rs_tau_counts."""
    def ok(t):
        return ~torch.isnan(t) if t.is_floating_point() else torch.ones_like(t, dtype=torch.bool)

    mx, my = ok(xt), ok(yt)
    both = mx & my

    def counts(a, b):
        if a.numel() < 2:
            return [0] * 6
        return tau_counts_device(a.contiguous(), b.contiguous()).cpu().tolist()

    c, d = counts(xt[both], yt[both])[:2]
    xs, ys = xt[mx], yt[my]
    n1 = counts(xs, xs)[2] + _pairs(n - xs.numel())
    n2 = counts(ys, ys)[3] + _pairs(n - ys.numel())
    return _finish(c, d, n1, n2, n)


# ---------------------------------------------------------------------------
# ListMLE
# ---------------------------------------------------------------------------


def _check_listmle_args(scores, true_order):
    s = np.asarray(scores, dtype=np.float64) if not isinstance(scores, torch.Tensor) else scores
    o = np.asarray(true_order, dtype=np.int64) if not isinstance(true_order, torch.Tensor) else true_order
    if len(s.shape) != 1 or tuple(o.shape) != tuple(s.shape):
        raise ValueError("scores and true_order must be equal-length 1-d arrays")
    return s, o


def list_mle_batched(scores: torch.Tensor, order: torch.Tensor):
    """[n_lists, L] scores (f32/f64) and int64 permutations -> (loss[n_lists], grad)."""
    if scores.dim() != 2 or order.shape != scores.shape:
        raise ValueError("scores and order must both be [n_lists, list_len]")
    dev = scores.device
    s = scores.contiguous()
    o = order.to(torch.int64).contiguous()
    n_lists, L = s.shape
    loss = torch.empty(n_lists, dtype=s.dtype, device=dev)
    grad = torch.empty_like(s)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    dt = _TORCH_DT[s.dtype]
    _lib.check(_lib.load().rs_listmle_order(s.data_ptr(), dt, o.data_ptr(), n_lists, L, loss.data_ptr(),
                                            grad.data_ptr(), bad.data_ptr(), _lib.stream_handle(dev)),
               "rs_listmle_order")
    return loss, grad, bad


def _listmle_single(scores, true_order):
    s, o = _check_listmle_args(scores, true_order)
    n = int(s.shape[0])
    if n == 0:
        return 0.0, np.zeros(0)
    dev = _lib.device()
    st = s.to(dev, torch.float64) if isinstance(s, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(s)).to(dev)
    ot = o.to(dev, torch.int64) if isinstance(o, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(o)).to(dev)
    loss, grad, bad = list_mle_batched(st.reshape(1, n), ot.reshape(1, n))
    if int(bad.item()):
        raise ValueError("true_order must be a permutation of 0..n-1")
    return float(loss.item()), grad.reshape(n).cpu().numpy()


def list_mle_loss(scores, true_order) -> float:
    """Plackett-Luce negative log-likelihood (drop-in for ranking.py:86-99)."""
    return _listmle_single(scores, true_order)[0]


def list_mle_gradient(scores, true_order) -> np.ndarray:
    """Gradient of list_mle_loss w.r.t. scores (drop-in for ranking.py:102-120)."""
    return _listmle_single(scores, true_order)[1]


def listmle_from_lengths(g: torch.Tensor, lengths: torch.Tensor, bucket_width: int = 10):
    """Training form: per list, order = stable argsort(lengths // width); returns
    (loss/L per list, dg = grad/L) as in predictors.py:379-384."""
    if bucket_width < 1:
        raise ValueError("bucket_width must be >= 1")
    if g.dim() != 2 or lengths.shape != g.shape:
        raise ValueError("g and lengths must both be [n_lists, list_len]")
    dev = g.device
    gf = g.to(torch.float32).contiguous()
    lt = lengths.to(torch.int32).contiguous()
    n_lists, L = gf.shape
    loss = torch.empty(n_lists, dtype=torch.float32, device=dev)
    dg = torch.empty_like(gf)
    _lib.check(_lib.load().rs_listmle_lengths(gf.data_ptr(), lt.data_ptr(), n_lists, L, bucket_width,
                                              loss.data_ptr(), dg.data_ptr(), _lib.stream_handle(dev)),
               "rs_listmle_lengths")
    return loss, dg


def bucket_lengths(lengths, bucket_width: int = 10):
    """label = length // width (drop-in for ranking.py:123-132)."""
    if bucket_width < 1:
        raise ValueError("bucket_width must be >= 1")
    if isinstance(lengths, torch.Tensor):
        return torch.div(lengths.to(torch.int64), bucket_width, rounding_mode="floor")
    arr = np.asarray(lengths, dtype=np.int64)
    return arr // bucket_width


__all__ = ["TauResult", "kendall_tau_b", "list_mle_loss", "list_mle_gradient", "bucket_lengths",
           "list_mle_batched", "listmle_from_lengths", "tau_counts_device", "tau_from_counts"]

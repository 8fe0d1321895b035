"""Ranking scheduling policy on the B200 (drop-in for ranksched.schedulers).

RankingPolicy.schedule keeps the reference contract (schedulers.py:219-240): it
takes the candidate Request objects and a KV budget, returns a BatchDecision(run,
promoted, demoted) and mutates starvation_count / priority / quantum on the passed
requests. The sort, greedy fill and starvation bump run in one rs_rank_step call over
an SoA image of the candidates; DeviceQueue keeps that SoA resident in HBM for the
fast path (no per-step Python gather).

Only the ranking policy is on the hot path; FCFS/SJF/SRTF/MLFQ stay the reference's
own (make_policy raises for them, install() delegates them to ranksched).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib

NS_PER_S = 1_000_000_000
UNLIMITED_KV = 1 << 62  # engine.py:39


@dataclass(frozen=True)
class SchedulerConfig:
    """Same fields, defaults and validation as schedulers.py:25-52."""

    max_batch: int = 256
    preemption: bool = True
    starvation_threshold: int = 100
    priority_quantum: int = 50
    mlfq_base_quantum: float = 16.0
    mlfq_growth: float = 2.0
    mlfq_num_queues: int = 8

    def __post_init__(self):
        if self.max_batch < 1:
            raise ValueError("max_batch must be >= 1")
        if self.starvation_threshold < 0:
            raise ValueError("starvation_threshold must be >= 0")
        if self.priority_quantum < 1:
            raise ValueError("priority_quantum must be >= 1")
        if self.mlfq_base_quantum <= 0 or self.mlfq_growth < 1:
            raise ValueError("bad MLFQ quantum parameters")
        if self.mlfq_num_queues < 1:
            raise ValueError("mlfq_num_queues must be >= 1")


@dataclass
class BatchDecision:
    run: list[int]
    promoted: list[int] = field(default_factory=list)
    demoted: list[int] = field(default_factory=list)


class DeviceQueue:
    """Resident SoA queue (A15 of SURVEY §8a) on one CUDA device.

    Rows are candidates in candidate order. Fields: score (f32 or f64), flags
    (scored/priority/running bits), prompt/generated tokens, arrival_rank, id,
    starvation, quantum — exactly the Request fields the ranking policy reads and
    writes (workload.py:40-61).
    """

    def __init__(self, n: int, dev: torch.device | None = None, score_dtype=torch.float64):
        dev = dev or _lib.device()
        self.dev = dev
        self.n = int(n)
        self.score = torch.zeros(n, dtype=score_dtype, device=dev)
        self.flags = torch.zeros(n, dtype=torch.uint8, device=dev)
        self.prompt_tokens = torch.ones(n, dtype=torch.int32, device=dev)
        self.generated_tokens = torch.zeros(n, dtype=torch.int32, device=dev)
        self.arrival_rank = torch.zeros(n, dtype=torch.int32, device=dev)
        self.id = torch.arange(n, dtype=torch.int64, device=dev)
        self.starvation = torch.zeros(n, dtype=torch.int32, device=dev)
        self.quantum = torch.zeros(n, dtype=torch.int32, device=dev)
        cap = max(self.n, 1)
        self.run_out = torch.empty(cap, dtype=torch.int64, device=dev)
        self.prom_out = torch.empty(cap, dtype=torch.int64, device=dev)
        self.dem_out = torch.empty(cap, dtype=torch.int64, device=dev)
        self.counts = torch.zeros(4, dtype=torch.int32, device=dev)

    @classmethod
    def from_arrays(cls, *, score, scored, priority, running, prompt_tokens, generated_tokens, arrival_time,
                    ids, starvation, quantum, dev=None, score_dtype=torch.float64):
        n = len(ids)
        q = cls(n, dev, score_dtype)
        d = q.dev

        def put(dst, src, dt):
            dst.copy_(torch.as_tensor(np.ascontiguousarray(src)).to(dt))

        put(q.score, score, score_dtype)
        fl = (np.asarray(scored, bool) * _lib.RS_FLAG_SCORED
              | np.asarray(priority, bool) * _lib.RS_FLAG_PRIORITY
              | np.asarray(running, bool) * _lib.RS_FLAG_RUNNING).astype(np.uint8)
        put(q.flags, fl, torch.uint8)
        put(q.prompt_tokens, prompt_tokens, torch.int32)
        put(q.generated_tokens, generated_tokens, torch.int32)
        put(q.id, ids, torch.int64)
        put(q.starvation, starvation, torch.int32)
        put(q.quantum, quantum, torch.int32)
        arr = torch.as_tensor(np.ascontiguousarray(np.asarray(arrival_time, dtype=np.float64))).to(d)
        q.set_arrival_rank(arr)
        return q

    def set_arrival_rank(self, arrival_time: torch.Tensor) -> None:
        """arrival_rank = position in (arrival_time, id) order, computed on the device."""
        lib = _lib.load()
        if self.n == 0:
            return
        ws, wn = _lib.workspace.get(lib.rs_arrival_rank_workspace_size(self.n), self.dev)
        _lib.check(lib.rs_arrival_rank(arrival_time.data_ptr(), self.id.data_ptr(), self.n,
                                       self.arrival_rank.data_ptr(), ws, wn, _lib.stream_handle(self.dev)),
                   "rs_arrival_rank")

    def soa(self) -> _lib.QueueSoA:
        return _lib.QueueSoA(
            self.n, _lib.RS_F32 if self.score.dtype == torch.float32 else _lib.RS_F64, self.score.data_ptr(),
            self.prompt_tokens.data_ptr(), self.generated_tokens.data_ptr(), self.arrival_rank.data_ptr(),
            self.id.data_ptr(), self.flags.data_ptr(), self.starvation.data_ptr(), self.quantum.data_ptr())

    def rank_step(self, config: SchedulerConfig, kv_budget: int | None, length_calibrated: bool,
                  preemptive: bool = True) -> None:
        """Enqueue one scheduling step (no host sync); results in run_out/prom_out/
        dem_out with counts[0:3] = (n_run, n_promoted, n_demoted), counts[3] = NaN flag."""
        lib = _lib.load()
        soa = self.soa()
        budget = -1 if kv_budget is None or kv_budget >= UNLIMITED_KV else int(kv_budget)
        ws, wn = _lib.workspace.get(lib.rs_rank_step_workspace_size(self.n), self.dev)
        if self.run_out.numel() < config.max_batch:
            self.run_out = torch.empty(config.max_batch, dtype=torch.int64, device=self.dev)
        _lib.check(lib.rs_rank_step(ctypes.byref(soa), config.max_batch, budget, config.starvation_threshold,
                                    config.priority_quantum, int(length_calibrated),
                                    int(preemptive and config.preemption), self.run_out.data_ptr(),
                                    self.prom_out.data_ptr(), self.dem_out.data_ptr(), self.counts.data_ptr(),
                                    ws, wn, _lib.stream_handle(self.dev)), "rs_rank_step")

    def rank_step_graph(self, config: SchedulerConfig, kv_budget: int | None, length_calibrated: bool,
                        preemptive: bool = True):
        """rank_step captured once as a CUDA graph for this queue (fixed n and buffers):
        returns a callable that replays it (one launch instead of ~20 at 1M rows)."""
        lib = _lib.load()
        ws = torch.empty(max(lib.rs_rank_step_workspace_size(self.n), 1), dtype=torch.uint8, device=self.dev)
        if self.run_out.numel() < config.max_batch:
            self.run_out = torch.empty(config.max_batch, dtype=torch.int64, device=self.dev)
        budget = -1 if kv_budget is None or kv_budget >= UNLIMITED_KV else int(kv_budget)
        soa = self.soa()

        def call():
            _lib.check(lib.rs_rank_step(ctypes.byref(soa), config.max_batch, budget, config.starvation_threshold,
                                        config.priority_quantum, int(length_calibrated),
                                        int(preemptive and config.preemption), self.run_out.data_ptr(),
                                        self.prom_out.data_ptr(), self.dem_out.data_ptr(), self.counts.data_ptr(),
                                        ws.data_ptr(), ws.numel(), _lib.stream_handle(self.dev)), "rs_rank_step")

        call()  # eager once (one-time kernel attributes), then capture
        torch.cuda.synchronize(self.dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            call()
        self._graph_keep = (g, ws, soa)
        return g.replay

    def decision(self) -> BatchDecision:
        c = self.counts.cpu().tolist()
        if c[3]:
            raise ValueError("ranking policy: NaN effective score")
        return BatchDecision(run=self.run_out[:c[0]].cpu().tolist(),
                             promoted=self.prom_out[:c[1]].cpu().tolist(),
                             demoted=self.dem_out[:c[2]].cpu().tolist())


class _Staging:
    """Grow-only pinned-host / device byte buffers holding one SoA image of the candidate
    list, so RankingPolicy.schedule moves its inputs with one H2D copy and its outputs
    with one D2H copy (no per-column transfers, no per-call allocations once warm)."""

    # (name, dtype, bytes per row); 16-byte aligned columns
    COLS = (("score", torch.float64, 8), ("arrival", torch.float64, 8), ("id", torch.int64, 8),
            ("prompt", torch.int32, 4), ("generated", torch.int32, 4), ("starvation", torch.int32, 4),
            ("quantum", torch.int32, 4), ("arrival_rank", torch.int32, 4), ("flags", torch.uint8, 1))
    OUTS = (("run", torch.int64, 8), ("prom", torch.int64, 8), ("dem", torch.int64, 8))

    def __init__(self, dev):
        self.dev, self.cap = dev, 0

    @staticmethod
    def _layout(cols, n):
        off, out = 0, {}
        for name, dt, w in cols:
            out[name] = (off, dt)
            off += -(-w * n // 16) * 16
        return out, off

    def ensure(self, n: int) -> None:
        """Room for n candidates (the run / promoted / demoted lists hold <= n ids)."""
        if n <= self.cap:
            return
        cap = max(n, 2 * self.cap, 1024)
        self.cap = cap
        self.in_lay, in_bytes = self._layout(self.COLS, cap)
        out_lay, out_bytes = self._layout(self.OUTS, cap)
        self.out_lay = {k: (o + in_bytes, dt) for k, (o, dt) in out_lay.items()}
        total = in_bytes + out_bytes + 16
        self.in_bytes = in_bytes
        self.host = torch.empty(total, dtype=torch.uint8).pin_memory()
        # zeroed once: the single D2H copy after a step also reads the unwritten tail of
        # the run / promoted / demoted slots (never consumed, but defined for initcheck)
        self.devbuf = torch.zeros(total, dtype=torch.uint8, device=self.dev)
        self.ws = torch.empty(max(_lib.load().rs_rank_step_workspace_size(cap),
                                  _lib.load().rs_arrival_rank_workspace_size(cap), 1),
                              dtype=torch.uint8, device=self.dev)

    def view(self, buf: torch.Tensor, name: str, n: int) -> torch.Tensor:
        off, dt = self.in_lay[name] if name in self.in_lay else self.out_lay[name]
        w = torch.empty((), dtype=dt).element_size()
        return buf[off:off + w * n].view(dt)


class RankingPolicy:
    """Score-ordered scheduling with starvation promotion (schedulers.py:178-240)."""

    name = "ranking"
    preemptive = True
    needs_scores = True
    decision_cls = BatchDecision  # install() substitutes the reference's BatchDecision

    def __init__(self, config: SchedulerConfig, length_calibrated: bool):
        self.config = config
        self.length_calibrated = length_calibrated
        self._stage: _Staging | None = None

    # host-side mirror of the reference key, kept for API compatibility (tests and
    # callers that sort with it); the scheduler itself sorts on the device.
    def effective_score(self, r) -> float:
        if r.score is None:
            return 0.0
        if self.length_calibrated:
            return r.score - r.generated_tokens
        return r.score

    def sort_key(self, r):
        return (0 if r.score is None else 1, 0 if r.priority else 1, self.effective_score(r),
                r.arrival_time, r.id)

    def on_admit(self, r) -> None:
        """Called once when the engine admits a request."""

    def record_execution(self, run, iter_ns: int) -> list[int]:
        return []

    def schedule(self, candidates, kv_budget: int) -> BatchDecision:
        """One ranking step over `candidates` (reference: schedulers.py:219-240 with
        Policy.schedule / _fill, :64-109): the AoS -> SoA gather is one pass over the
        Request objects into a pinned staging image, one H2D copy, rs_arrival_rank +
        rs_rank_step on the device, one D2H copy of decision and state, and the mutated
        starvation_count / priority / quantum written back to the passed requests."""
        cands = candidates if isinstance(candidates, list) else list(candidates)
        n = len(cands)
        if n == 0:
            return self.decision_cls(run=[])
        dev = _lib.device()
        if self._stage is None or self._stage.dev != dev:
            self._stage = _Staging(dev)
        stg = self._stage
        stg.ensure(n)
        h = stg.host
        rows = [(r.score, r.arrival_time, r.id, r.prompt_tokens, r.generated_tokens, r.starvation_count,
                 r.quantum, r.priority, r.state) for r in cands]
        sc, arr, ids, pt, gt, stv, qu, pr, st = zip(*rows)
        scored = np.fromiter((v is not None for v in sc), bool, n)
        score = np.fromiter((0.0 if v is None else v for v in sc), np.float64, n)
        running = np.fromiter((getattr(v, "value", v) == "running" for v in st), bool, n)
        priority = np.fromiter(pr, bool, n)
        stg.view(h, "score", n).numpy()[:] = score
        stg.view(h, "arrival", n).numpy()[:] = arr
        stg.view(h, "id", n).numpy()[:] = ids
        stg.view(h, "prompt", n).numpy()[:] = pt
        stg.view(h, "generated", n).numpy()[:] = gt
        stv_old = np.asarray(stv, dtype=np.int64)
        qu_old = np.asarray(qu, dtype=np.int64)
        stg.view(h, "starvation", n).numpy()[:] = stv_old
        stg.view(h, "quantum", n).numpy()[:] = qu_old
        stg.view(h, "flags", n).numpy()[:] = (scored * _lib.RS_FLAG_SCORED | priority * _lib.RS_FLAG_PRIORITY
                                             | running * _lib.RS_FLAG_RUNNING)
        d = stg.devbuf
        stream = _lib.stream_handle(dev)
        d[:stg.in_bytes].copy_(h[:stg.in_bytes], non_blocking=True)
        lib = _lib.load()
        V = lambda name: stg.view(d, name, n).data_ptr()  # noqa: E731
        _lib.check(lib.rs_arrival_rank(V("arrival"), V("id"), n, V("arrival_rank"), stg.ws.data_ptr(),
                                       stg.ws.numel(), stream), "rs_arrival_rank")
        soa = _lib.QueueSoA(n, _lib.RS_F64, V("score"), V("prompt"), V("generated"), V("arrival_rank"), V("id"),
                            V("flags"), V("starvation"), V("quantum"))
        cnt_off = d.numel() - 16
        counts = d[cnt_off:cnt_off + 16].view(torch.int32)
        budget = -1 if kv_budget is None or kv_budget >= UNLIMITED_KV else int(kv_budget)
        _lib.check(lib.rs_rank_step(ctypes.byref(soa), self.config.max_batch, budget,
                                    self.config.starvation_threshold, self.config.priority_quantum,
                                    int(self.length_calibrated), int(self.preemptive and self.config.preemption),
                                    V("run"), V("prom"), V("dem"), counts.data_ptr(), stg.ws.data_ptr(),
                                    stg.ws.numel(), stream), "rs_rank_step")
        # one D2H copy: the mutated state columns through the end of the buffer
        lo = stg.in_lay["starvation"][0]
        h[lo:].copy_(d[lo:], non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        c = h[cnt_off:cnt_off + 16].view(torch.int32).tolist()
        if c[3]:
            raise ValueError("ranking policy: NaN effective score")
        dec = self.decision_cls(run=stg.view(h, "run", c[0]).tolist(), promoted=stg.view(h, "prom", c[1]).tolist(),
                                demoted=stg.view(h, "dem", c[2]).tolist())
        fl = stg.view(h, "flags", n).numpy()
        pr_new = (fl & _lib.RS_FLAG_PRIORITY) != 0
        stv_new = stg.view(h, "starvation", n).numpy().tolist()
        qu_new = stg.view(h, "quantum", n).numpy().tolist()
        for k, r in enumerate(cands):
            r.starvation_count = stv_new[k]
            r.quantum = qu_new[k]
        for k in np.nonzero(pr_new != priority)[0].tolist():
            cands[k].priority = bool(pr_new[k])
        return dec


def make_policy(name: str, config: SchedulerConfig, length_calibrated: bool = True):
    """Factory (schedulers.py:243-256) for the policy on the B200 hot path."""
    name = name.lower()
    if name == "ranking":
        return RankingPolicy(config, length_calibrated)
    if name in ("fcfs", "sjf", "srtf", "mlfq"):
        raise ValueError(f"policy {name!r} is a baseline outside the B200 hot path; "
                         "use ranksched.schedulers.make_policy (install() wires both)")
    raise ValueError(f"unknown policy {name!r}")

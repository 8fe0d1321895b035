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
from .workload import is_running

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


class RankingPolicy:
    """Score-ordered scheduling with starvation promotion (schedulers.py:178-240)."""

    name = "ranking"
    preemptive = True
    needs_scores = True

    def __init__(self, config: SchedulerConfig, length_calibrated: bool):
        self.config = config
        self.length_calibrated = length_calibrated

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
        cands = list(candidates)
        n = len(cands)
        if n == 0:
            return BatchDecision(run=[])
        scored = [r.score is not None for r in cands]
        q = DeviceQueue.from_arrays(
            score=[r.score if r.score is not None else 0.0 for r in cands], scored=scored,
            priority=[bool(r.priority) for r in cands], running=[is_running(r) for r in cands],
            prompt_tokens=[r.prompt_tokens for r in cands], generated_tokens=[r.generated_tokens for r in cands],
            arrival_time=[r.arrival_time for r in cands], ids=[r.id for r in cands],
            starvation=[r.starvation_count for r in cands], quantum=[r.quantum for r in cands])
        q.rank_step(self.config, kv_budget, self.length_calibrated, self.preemptive)
        dec = q.decision()
        flags = q.flags.cpu().numpy()
        starv = q.starvation.cpu().tolist()
        quant = q.quantum.cpu().tolist()
        for k, r in enumerate(cands):
            r.priority = bool(flags[k] & _lib.RS_FLAG_PRIORITY)
            r.starvation_count = starv[k]
            r.quantum = quant[k]
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

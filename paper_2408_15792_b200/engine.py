"""Device-resident scheduler loop: the reference's `engine.run` (engine.py:382-460) for
the ranking policy, with the queue, the policy state and the latency bookkeeping in HBM.

SURVEY §8f #1 / BASELINE.json configs[4]. Per step, exactly as the reference:
`jump_if_idle` / `admit_due` (engine.py:218-243; admission and the KV drop rule are
host decisions on the sorted arrival times), scoring of the newly admitted requests
(charged `predictor_ns_per_request` once each when the scorer `charges_predictor`),
`RankingPolicy.schedule` (rs_rank_step), `_Sim.execute` (rs_engine_execute) and the
step record. Scores come from a per-request score cache: the OPT ranker is a pure
function of the prompt, so scoring every request once up front — batched
on the GPU(s) — gives the same scores `rescore=True` would recompute every step, and
the reference charges predictor time only at the first scoring either way.

Records, per-request rows and metrics use the reference's keys and arithmetic (integer
nanoseconds, math.fsum means, nearest-rank p90), so a run can be compared bit for bit
with `ranksched.engine.run(trace, "ranking", scorer)` on the same scores
(tests/test_gpu_engine.py, against fixtures recorded from the reference). Record-free
runs execute the whole loop as one device launch (csrc/rankstep.cu engine_loop_kernel;
tests/test_gpu_engine_loop.py checks it against the per-step path).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import asdict, dataclass, field

import numpy as np
import torch

from . import _lib
from .schedulers import SchedulerConfig, UNLIMITED_KV

NS_PER_S = 1_000_000_000


@dataclass(frozen=True)
class CostModel:
    """Iteration timing in nanoseconds (the reference's CostModel, engine.py:42-78)."""

    decode_ns: int = 25_000_000
    prefill_ns_per_token: int = 40_000
    predictor_ns_per_request: int = 500_000
    decode_table: tuple[int, ...] | None = None

    def __post_init__(self):
        if self.decode_ns <= 0:
            raise ValueError("decode_ns must be > 0")
        if self.prefill_ns_per_token < 0 or self.predictor_ns_per_request < 0:
            raise ValueError("cost components must be >= 0")
        if self.decode_table is not None:
            object.__setattr__(self, "decode_table", tuple(self.decode_table))
            if not self.decode_table or any(v <= 0 for v in self.decode_table):
                raise ValueError("decode_table entries must be > 0")


COST_PRESETS = {
    "default": CostModel(),
    "fast": CostModel(decode_ns=1_000_000, prefill_ns_per_token=2_000, predictor_ns_per_request=20_000),
    "unit": CostModel(decode_ns=NS_PER_S, prefill_ns_per_token=0, predictor_ns_per_request=0),
}


@dataclass
class EngineResult:
    metrics: dict
    requests: list[dict]
    records: list[dict] = field(default_factory=list, repr=False)
    steps: int = 0


def _p90(values):
    s = sorted(values)
    return s[math.ceil(0.9 * len(s)) - 1]


def _latency_stats(lat, ptl, mw, makespan):
    """ranking.latency_stats (ranking.py:167-201): fsum means, nearest-rank p90."""
    n = len(lat)
    if n == 0:
        return dict(mean_latency=0.0, p90_latency=0.0, mean_per_token_latency=0.0, p90_per_token_latency=0.0,
                    throughput=0.0, mean_max_waiting_time=0.0, p90_max_waiting_time=0.0, makespan=float(makespan))
    return dict(mean_latency=math.fsum(lat) / n, p90_latency=_p90(lat), mean_per_token_latency=math.fsum(ptl) / n,
                p90_per_token_latency=_p90(ptl), throughput=n / makespan if makespan > 0 else 0.0,
                mean_max_waiting_time=math.fsum(mw) / n, p90_max_waiting_time=_p90(mw), makespan=float(makespan))


class DeviceEngine:
    """One simulation of a trace under the ranking policy, state resident on `dev`."""

    def __init__(self, requests, scores, sched: SchedulerConfig = SchedulerConfig(),
                 cost: CostModel = COST_PRESETS["default"], kv_budget: int | None = None,
                 length_calibrated: bool = False, charges_predictor: bool = True, dev=None,
                 in_place_compaction: bool = False):
        self.reqs = list(requests)
        n = len(self.reqs)
        if len(scores) != n:
            raise ValueError("one score per request")
        self.sched, self.cost = sched, cost
        self.kv_budget = UNLIMITED_KV if kv_budget is None else int(kv_budget)
        if self.kv_budget < 1:
            raise ValueError("kv_budget must be >= 1")
        self.length_calibrated = bool(length_calibrated)
        self.charges_predictor = bool(charges_predictor)
        self.dev = dev or _lib.device()
        d = self.dev
        self.ids = np.array([r.id for r in self.reqs], dtype=np.int64)
        arr_s = [r.arrival_time for r in self.reqs]
        if any(b < a for a, b in zip(arr_s, arr_s[1:])):
            raise ValueError("trace requests not sorted by arrival_time")
        self.arrival_ns = np.array([int(round(t * NS_PER_S)) for t in arr_s], dtype=np.int64)
        self.prompt = np.array([r.prompt_tokens for r in self.reqs], dtype=np.int32)
        self.true_out = np.array([r.true_output_tokens for r in self.reqs], dtype=np.int32)
        # arrival rank: position in (arrival_time, id) order (the sort key's tail)
        order = np.lexsort((self.ids, np.array(arr_s, dtype=np.float64)))
        rank = np.empty(n, dtype=np.uint32)
        rank[order] = np.arange(n, dtype=np.uint32)
        sc = np.asarray(scores, dtype=np.float64)
        if np.isnan(sc).any():
            raise ValueError("ranking policy: NaN score")
        i32, i64 = torch.int32, torch.int64
        self.t_score = torch.from_numpy(sc).to(d)
        self.t_prompt = torch.from_numpy(self.prompt).to(d)
        self.t_true = torch.from_numpy(self.true_out).to(d)
        self.t_rank = torch.from_numpy(rank.view(np.int32)).to(d)
        self.t_arr = torch.from_numpy(self.arrival_ns).to(d)
        self.row_of = torch.full((n,), -1, dtype=i32, device=d)
        self.stamp = torch.full((n,), -1, dtype=i32, device=d)
        self.first_tok = torch.full((n,), -1, dtype=i64, device=d)
        self.last_ev = torch.zeros(n, dtype=i64, device=d)
        self.max_gap = torch.zeros(n, dtype=i64, device=d)
        self.finish = torch.full((n,), -1, dtype=i64, device=d)
        self.n_pre = torch.zeros(n, dtype=i32, device=d)
        cap = max(n, 1)
        # Queue columns. Out-of-place compaction (the default) keeps two column sets and
        # swaps them every step: execute compacts the survivors of set `cur` into the other
        # set with many CTAs (rs_engine_execute_ex); in place, one CTA does it (the
        # rs_engine_execute path, kept selectable for tests).
        self.in_place = bool(in_place_compaction)
        self._sets = []
        for _ in range(1 if self.in_place else 2):
            self._sets.append({
                "score": torch.zeros(cap, dtype=torch.float64, device=d),
                "flags": torch.zeros(cap, dtype=torch.uint8, device=d),
                "prompt": torch.zeros(cap, dtype=i32, device=d), "gen": torch.zeros(cap, dtype=i32, device=d),
                "rank": torch.zeros(cap, dtype=i32, device=d), "id": torch.zeros(cap, dtype=i64, device=d),
                "starv": torch.zeros(cap, dtype=i32, device=d), "quant": torch.zeros(cap, dtype=i32, device=d)})
        self.compact_scratch = torch.zeros((cap + 1023) // 1024 + 1, dtype=i32, device=d)
        # the previous step's batch (rs_engine_execute_ex's prev_run / prev_n)
        self.prev_run = torch.zeros(max(sched.max_batch, 1), dtype=i64, device=d)
        self.prev_n = torch.zeros(1, dtype=i32, device=d)
        self.run_out = torch.empty(max(sched.max_batch, 1), dtype=i64, device=d)
        self.prom_out = torch.empty(cap, dtype=i64, device=d)
        self.dem_out = torch.empty(cap, dtype=i64, device=d)
        self.pre_out = torch.empty(cap, dtype=i64, device=d)
        self.fin_out = torch.empty(max(sched.max_batch, 1), dtype=i64, device=d)
        # one 64-byte status block per step: out int64[6] (execute) | counts int32[4] (rank step),
        # read back with a single D2H copy
        self.stat = torch.zeros(8, dtype=i64, device=d)
        self.out = self.stat[:6]
        self.counts = self.stat[6:].view(i32)
        self.stat_host = torch.zeros(8, dtype=i64).pin_memory()
        self.out_host = self.stat_host[:6]
        self.cnt_host = self.stat_host[6:].view(i32)
        self.adm_host = torch.zeros(cap, dtype=i32).pin_memory()
        self.adm_dev = torch.zeros(cap, dtype=i32, device=d)
        dt = cost.decode_table
        self.t_table = torch.tensor(dt, dtype=i64, device=d) if dt else None
        self._trace = _lib.EngineTrace(self.t_score.data_ptr(), self.t_prompt.data_ptr(), self.t_true.data_ptr(),
                                       self.t_rank.data_ptr(), self.t_arr.data_ptr(), self.row_of.data_ptr(),
                                       self.stamp.data_ptr(), self.first_tok.data_ptr(), self.last_ev.data_ptr(),
                                       self.max_gap.data_ptr(), self.finish.data_ptr(), self.n_pre.data_ptr())
        self._cost = _lib.EngineCost(cost.decode_ns, cost.prefill_ns_per_token,
                                     None if self.t_table is None else self.t_table.data_ptr(),
                                     0 if dt is None else len(dt))

    @staticmethod
    def _cols(c):
        return (c["score"].data_ptr(), c["prompt"].data_ptr(), c["gen"].data_ptr(), c["rank"].data_ptr(),
                c["id"].data_ptr(), c["flags"].data_ptr(), c["starv"].data_ptr(), c["quant"].data_ptr())

    def _queue(self, n_alive: int, which: int = 0) -> _lib.EngineQueue:
        return _lib.EngineQueue(n_alive, _lib.RS_F64, *self._cols(self._sets[which]))

    def _soa(self, n_alive: int, which: int = 0) -> _lib.QueueSoA:
        return _lib.QueueSoA(n_alive, _lib.RS_F64, *self._cols(self._sets[which]))

    def run(self, record: bool = False, stop_after_finished: int | None = None,
            time_limit_s: float | None = None, native: bool = True, rescore=None,
            max_steps: int | None = None) -> EngineResult:
        """record=False (and native) runs the whole loop natively (rs_engine_run: with an
        unlimited KV budget one cluster launch steps the queue on the device, else a C++
        host loop over the per-step kernels); record=True steps from Python so every
        step's decision can be read back. rescore (optional):
        called every step with the alive requests' trace indices (int64 device tensor, queue
        order) and returning their scores (float64 device tensor): the reference's
        re-score-every-step mode (engine.py:414-428 with rescore=True) instead of the cache."""
        if native and not record and not self.in_place and rescore is None and max_steps is None:
            return self._run_native(stop_after_finished, time_limit_s)
        lib = _lib.load()
        rank_step, execute, admit, check = lib.rs_rank_step, lib.rs_engine_execute, lib.rs_engine_admit, _lib.check
        st = _lib.stream_handle(self.dev)
        stream = torch.cuda.current_stream(self.dev)
        n = len(self.reqs)
        limit_ns = None if time_limit_s is None else int(round(time_limit_s * NS_PER_S))
        sched = self.sched
        budget = -1 if self.kv_budget >= UNLIMITED_KV else self.kv_budget
        fits = (self.prompt.astype(np.int64) + self.true_out) <= self.kv_budget
        nsets = len(self._sets)
        qs = [self._queue(0, i) for i in range(nsets)]
        soas = [self._soa(0, i) for i in range(nsets)]
        q_refs = [ctypes.byref(x) for x in qs]
        soa_refs = [ctypes.byref(x) for x in soas]
        tr_ref, cost_ref = ctypes.byref(self._trace), ctypes.byref(self._cost)
        execute_ex = lib.rs_engine_execute_ex
        scratch_p = self.compact_scratch.data_ptr()
        self.prev_n.zero_()
        prev_run_p, prev_n_p = self.prev_run.data_ptr(), self.prev_n.data_ptr()
        cur = 0
        run_p, prom_p, dem_p, cnt_p = (self.run_out.data_ptr(), self.prom_out.data_ptr(), self.dem_out.data_ptr(),
                                       self.counts.data_ptr())
        out_p, pre_p, fin_p, adm_p = (self.out.data_ptr(), self.pre_out.data_ptr(), self.fin_out.data_ptr(),
                                      self.adm_dev.data_ptr())
        adm_np = self.adm_host.numpy()
        out_np, cnt_np = self.out_host.numpy(), self.cnt_host.numpy()
        ws_n = 0
        ws = wn = None
        now, nxt, n_alive, step, n_finished = 0, 0, 0, 0, 0
        dev_now = None  # the device copy of the clock (out[0]) when known to equal `now`
        # loop-invariant values and bound methods, hoisted (the loop runs ~10^5 times)
        arr_list = self.arrival_ns.tolist()
        pred_ns_per_req = self.cost.predictor_ns_per_request if self.charges_predictor else 0
        max_batch, threshold, quantum = sched.max_batch, sched.starvation_threshold, sched.priority_quantum
        calibrated, preemptive = int(self.length_calibrated), int(sched.preemption)
        stat_host_copy, stat_dev, sync = self.stat_host.copy_, self.stat, stream.synchronize
        tot_prefill = tot_decode = tot_pred = 0
        dropped_all: list[int] = []
        records = []
        while True:
            if n_alive == 0 and nxt < n and arr_list[nxt] > now:  # jump_if_idle
                now = arr_list[nxt]
            # admit_due: the arrivals up to `now`; requests that could never hold their
            # full context in the KV budget are dropped (engine.py:224-243)
            end = nxt  # arrivals are sorted and few per step: walk instead of bisecting
            while end < n and arr_list[end] <= now:
                end += 1
            admitted = dropped = None
            k = 0
            if end > nxt:
                idx = np.arange(nxt, end)
                ok = fits[nxt:end]
                admitted, dropped = idx[ok], idx[~ok]
                nxt = end
                k = len(admitted)
                if len(dropped):
                    dropped_all.extend(dropped.tolist())
                if k:
                    adm_np[:k] = admitted
                    self.adm_dev[:k].copy_(self.adm_host[:k], non_blocking=True)
                    qs[cur].n = n_alive
                    check(admit(q_refs[cur], tr_ref, adm_p, k, n_alive, st), "rs_engine_admit")
                    n_alive += k
            if n_alive == 0:
                break
            if limit_ns is not None and now >= limit_ns:
                break
            predictor_ns = k * pred_ns_per_req
            if n_alive > ws_n:
                ws_n = max(n_alive, 2 * ws_n)
                ws, wn = self._rank_workspace(lib.rs_rank_step_workspace_size(ws_n))
            if rescore is not None:
                cols = self._sets[cur]
                cols["score"][:n_alive].copy_(rescore(cols["id"][:n_alive]))
            soas[cur].n = n_alive
            rc = rank_step(soa_refs[cur], max_batch, budget, threshold, quantum, calibrated, preemptive, run_p, prom_p,
                           dem_p, cnt_p, ws, wn, st)
            if rc:
                check(rc, "rs_rank_step")
            if now != dev_now:  # the clock moved on the host (idle jump / first step)
                out_np[0] = now
                self.out[:1].copy_(self.out_host[:1], non_blocking=True)
                dev_now = now
            qs[cur].n = n_alive
            if nsets == 1:
                check(execute(q_refs[0], tr_ref, cost_ref, run_p, cnt_p, step, predictor_ns, out_p, pre_p, fin_p, st),
                      "rs_engine_execute")
            else:
                rc = execute_ex(q_refs[cur], q_refs[1 - cur], tr_ref, cost_ref, run_p, cnt_p, step, predictor_ns,
                                out_p, pre_p, fin_p, scratch_p, prev_run_p, prev_n_p, st)
                if rc:
                    check(rc, "rs_engine_execute_ex")
                cur = 1 - cur
            stat_host_copy(stat_dev, non_blocking=True)
            sync()
            if cnt_np[3]:
                raise ValueError("ranking policy: NaN effective score")
            now, iter_ns, prefill_ns, n_alive = int(out_np[0]), int(out_np[1]), int(out_np[2]), int(out_np[3])
            dev_now = now
            n_finished += int(out_np[5])
            tot_prefill += prefill_ns
            tot_pred += predictor_ns
            tot_decode += iter_ns - prefill_ns - predictor_ns
            if record:
                ids, c = self.ids, cnt_np.tolist()
                adm = [] if admitted is None else ids[admitted].tolist()
                records.append({
                    "step": step, "now_ns": now, "iter_ns": iter_ns,
                    "run": ids[self.run_out[:c[0]].cpu().numpy()].tolist(),
                    "preempted": ids[self.pre_out[:int(out_np[4])].cpu().numpy()].tolist(),
                    "promoted": ids[self.prom_out[:c[1]].cpu().numpy()].tolist(),
                    "demoted": ids[self.dem_out[:c[2]].cpu().numpy()].tolist(),
                    "admitted": adm, "dropped": [] if dropped is None else ids[dropped].tolist(),
                    "finished": ids[self.fin_out[:int(out_np[5])].cpu().numpy()].tolist(),
                    "scored": adm, "predictor_ns": predictor_ns,
                })
            step += 1
            if stop_after_finished is not None and n_finished >= stop_after_finished:
                break
            if max_steps is not None and step >= max_steps:
                break
            if limit_ns is not None and now >= limit_ns:
                break
        rows = self._rows(set(dropped_all), nxt)
        metrics = self._metrics(rows, now, step)
        metrics.update(total_prefill_ns=tot_prefill, total_decode_ns=tot_decode, total_predictor_ns=tot_pred)
        return EngineResult(metrics, rows, records, step)

    def _rank_workspace(self, nbytes: int) -> tuple[int, int]:
        """The engine's own rank-step scratch (grow-only). Not the shared per-device
        workspace: a rescore() callback may grow that one mid-run and free the buffer
        whose address the loop holds."""
        buf = getattr(self, "_rank_ws", None)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(int(nbytes), 1 << 20), dtype=torch.uint8, device=self.dev)
            self._rank_ws = buf
        return buf.data_ptr(), buf.numel()

    def _run_native(self, stop_after_finished, time_limit_s) -> EngineResult:
        lib = _lib.load()
        n = len(self.reqs)
        q2 = (_lib.EngineQueue * 2)(self._queue(0, 0), self._queue(0, 1))
        soa2 = (_lib.QueueSoA * 2)(self._soa(0, 0), self._soa(0, 1))
        fits = np.ascontiguousarray(((self.prompt.astype(np.int64) + self.true_out) <= self.kv_budget).astype(np.uint8))
        arr = np.ascontiguousarray(self.arrival_ns, dtype=np.int64)
        dropped = np.empty(max(n, 1), dtype=np.int64)
        ws, wn = self._rank_workspace(lib.rs_rank_step_workspace_size(max(n, 1)))
        sched = self.sched
        self.prev_n.zero_()
        lp = _lib.EngineLoop(
            n, arr.ctypes.data, fits.ctypes.data, self.adm_host.data_ptr(), self.adm_dev.data_ptr(),
            dropped.ctypes.data, self.stat.data_ptr(), self.stat_host.data_ptr(), self.run_out.data_ptr(),
            self.prom_out.data_ptr(), self.dem_out.data_ptr(), self.pre_out.data_ptr(), self.fin_out.data_ptr(),
            self.compact_scratch.data_ptr(), self.prev_run.data_ptr(), self.prev_n.data_ptr(), ws, wn,
            sched.max_batch, sched.starvation_threshold,
            sched.priority_quantum, int(self.length_calibrated), int(sched.preemption),
            -1 if self.kv_budget >= UNLIMITED_KV else self.kv_budget,
            self.cost.predictor_ns_per_request if self.charges_predictor else 0,
            -1 if time_limit_s is None else int(round(time_limit_s * NS_PER_S)),
            -1 if stop_after_finished is None else int(stop_after_finished))
        out = _lib.EngineLoopOut()
        rc = lib.rs_engine_run(q2, soa2, ctypes.byref(self._trace), ctypes.byref(self._cost), ctypes.byref(lp),
                               ctypes.byref(out), _lib.stream_handle(self.dev))
        if rc == _lib.RS_ERR_NAN:
            raise ValueError("ranking policy: NaN effective score")
        _lib.check(rc, "rs_engine_run")
        rows = self._rows(set(dropped[:out.n_dropped].tolist()), out.next_arrival)
        metrics = self._metrics(rows, out.now_ns, out.steps)
        metrics.update(total_prefill_ns=out.total_prefill_ns, total_decode_ns=out.total_decode_ns,
                       total_predictor_ns=out.total_predictor_ns)
        return EngineResult(metrics, rows, [], out.steps)

    def _rows(self, dropped: set[int], n_arrived: int) -> list[dict]:
        first = self.first_tok.cpu().numpy()
        fin = self.finish.cpu().numpy()
        gap = self.max_gap.cpu().numpy()
        npre = self.n_pre.cpu().numpy()
        rows = []
        for i, r in enumerate(self.reqs):
            arrived = i < n_arrived
            if i in dropped:
                status = "dropped"
            elif not arrived:
                status = "unarrived"
            elif fin[i] >= 0:
                status = "finished"
            else:
                status = "unfinished"
            row = {"id": r.id, "arrival_s": r.arrival_time, "prompt_tokens": r.prompt_tokens,
                   "output_tokens": r.true_output_tokens, "status": status, "first_token_s": None, "finish_s": None,
                   "latency_s": None, "per_token_latency_s": None, "max_wait_s": None,
                   "n_preempted": int(npre[i]) if arrived and i not in dropped else 0}
            if arrived and first[i] >= 0:
                row["first_token_s"] = int(first[i]) / NS_PER_S
                row["max_wait_s"] = int(gap[i]) / NS_PER_S
            if arrived and fin[i] >= 0:
                row["finish_s"] = int(fin[i]) / NS_PER_S
                lat_ns = int(fin[i]) - int(self.arrival_ns[i])
                row["latency_s"] = lat_ns / NS_PER_S
                row["per_token_latency_s"] = lat_ns / r.true_output_tokens / NS_PER_S
            rows.append(row)
        return rows

    def _metrics(self, rows: list[dict], now_ns: int, steps: int) -> dict:
        from .ranking import kendall_tau_b
        done = [r for r in rows if r["status"] == "finished"]
        stats = _latency_stats([r["latency_s"] for r in done], [r["per_token_latency_s"] for r in done],
                               [r["max_wait_s"] for r in done], now_ns / NS_PER_S)
        tau = kendall_tau_b([r["first_token_s"] for r in done], [r["output_tokens"] for r in done]).tau \
            if len(done) >= 2 else 0.0
        return {"n_finished": len(done), "n_dropped": sum(1 for r in rows if r["status"] == "dropped"),
                "n_unfinished": sum(1 for r in rows if r["status"] in ("unfinished", "unarrived")),
                "n_preemptions": sum(r["n_preempted"] for r in rows), "steps": steps,
                "makespan_s": stats["makespan"], "throughput_rps": stats["throughput"],
                "mean_latency_s": stats["mean_latency"], "p90_latency_s": stats["p90_latency"],
                "mean_per_token_latency_s": stats["mean_per_token_latency"],
                "p90_per_token_latency_s": stats["p90_per_token_latency"],
                "mean_max_waiting_s": stats["mean_max_waiting_time"],
                "p90_max_waiting_s": stats["p90_max_waiting_time"], "execution_order_tau": tau}


def run(trace, scorer=None, scores=None, sched: SchedulerConfig = SchedulerConfig(),
        cost: CostModel = COST_PRESETS["default"], kv_budget: int | None = None, seed: int = 0,
        record: bool = False, stop_after_finished: int | None = None, time_limit_s: float | None = None,
        in_place_compaction: bool = False):
    """engine.run(trace, "ranking", scorer, ...) on the device. Give either a scorer (its
    score_batch is called once over the whole trace: the score cache) or `scores`."""
    reqs = list(trace)
    if scores is None:
        if scorer is None:
            raise ValueError("policy 'ranking' needs a scorer")
        scores = scorer.score_batch(reqs, seed) if reqs else []
        if any(s is None for s in scores):
            raise ValueError("the device engine needs a score for every request (warm-up scorers unsupported)")
    length_calibrated = getattr(scorer, "length_calibrated", False) if scorer is not None else False
    charges = getattr(scorer, "charges_predictor", True) if scorer is not None else True
    eng = DeviceEngine(reqs, scores, sched, cost, kv_budget, length_calibrated, charges,
                       in_place_compaction=in_place_compaction)
    return eng.run(record=record, stop_after_finished=stop_after_finished, time_limit_s=time_limit_s)

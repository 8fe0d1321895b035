#!/usr/bin/env python
"""Benchmark: prompts ranked/sec (OPT-125M-shape score + sort) on B200; tau pairs/sec.

Workload (BASELINE.json configs[1]): every rank scores 4096 synthetic prompts x 512
token ids with the random-init OPT-125M-shape ranker (bf16 GEMM operands, fp32
accumulate / residual), the scores are all-gathered to rank 0 (NCCL, the only
collective), and rank 0 runs the ranking-policy step (sort + fill + starvation
bump, max_batch 256) over the global batch. One step = that whole pass; value =
prompts of all ranks / max-over-ranks device time. Scaling is weak (4096 prompts
per GPU). Secondary lines in the same JSON: tau pairs/s and rank-step requests/s on
the 1M-request cfg4 queue (BASELINE.json configs[3]).

    python bench.py [--gpus N --steps K --warmup W]           # our B200 path
    python bench.py --impl reference ...                      # CPU oracle port arm
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import time

import numpy as np
import torch

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "prompts ranked/sec (OPT-125M score+sort) at 1/2/4/8 B200; tau pairs/sec"
UNIT = "prompts/s"
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        d["source"] = "measured (MEASURED_PEAKS.json)"
        return d
    d = dict(FALLBACK_PEAKS)
    d["source"] = "fallback (B200_PROFILING.md)"
    return d


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md recipe)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out = ""

    def summary(self):
        rows = [r.split(",") for r in self.out.strip().splitlines() if r.count(",") >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].strip() == "Active"})
        loaded = [s for s in sm if mx and s > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(rows), "reasons": reasons}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_cores():
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


# ---------------------------------------------------------------------------
# CPU baselines (bench_cpu.py) and the --impl reference arm
# ---------------------------------------------------------------------------


def cpu_baseline(cfg, S, n_prompts=16):
    import bench_cpu
    return bench_cpu.headline(cfg, S, n_prompts)


def run_reference(args):
    """The reference arm: the CPU path timed on the host cores, each step a bounded sample
    of the headline workload (bench_cpu.HeadlineCPU: fp32 OPT forward port on all threads —
    the reference has no OPT model — + the reference's own RankingPolicy.schedule)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import bench_cpu
    from paper_2408_15792_b200.ranker import RankerConfig
    cfg = RankerConfig.opt_125m()
    P = args.ref_prompts
    h = bench_cpu.HeadlineCPU(cfg, args.seq, P)
    for _ in range(args.warmup):
        h.step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        h.step()
    dt = (time.perf_counter() - t0) / args.steps
    v = P / dt
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (random token ids, random-init weights, seed 0)",
            "config": {"workload": f"OPT-125M-shape ranker scoring {args.batch} prompts x {args.seq} tokens + score "
                                   f"sort; each CPU step is a bounded sample of {P} prompts",
                       "global_batch": args.batch, "seq_len": args.seq, "parallelism": "cpu"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": h.torch.get_num_threads(), "kind": h.kind,
                             "sample": h.describe(dt)},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# B200 path
# ---------------------------------------------------------------------------


def timed(fn, reps, stream=None):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def gemm_roofline(pk, M=1 << 20, reps=5):
    """Per-launch CUDA-event timing of the four projection GEMMs at the forward's
    chunk shape; achieved = algorithmic FLOPs per launch / average launch time."""
    from paper_2408_15792_b200 import _lib
    lib = _lib.load()
    shapes = [(2304, 768, 7), (768, 768, 2), (3072, 768, 1), (768, 3072, 2)]
    res = []
    tot_f = tot_t = 0.0
    for N, K, epi in shapes:
        A = torch.randn(M, K, device="cuda").bfloat16()
        W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
        b = torch.zeros(N, device="cuda").bfloat16()
        C = torch.empty(M, N, device="cuda", dtype=torch.float32 if epi == 2 else torch.bfloat16)
        R = C if epi == 2 else None

        def f():
            _lib.check(lib.rs_gemm_bf16(A.data_ptr(), W.data_ptr(), b.data_ptr(), None if R is None else R.data_ptr(),
                                        C.data_ptr(), M, N, K, epi, _lib.stream_handle()))
        f()
        t = timed(f, reps)
        fl = 2.0 * M * N * K
        res.append({"N": N, "K": K, "ms": t, "tflops": fl / t / 1e9})
        tot_f += fl
        tot_t += t
        del A, W, C
    achieved = tot_f / tot_t / 1e9
    # DRAM bytes of the same four launches from the committed ncu --set full capture
    traffic = None
    tp = ROOT / "profiles" / "r02_gemm_traffic.json"
    if not tp.exists():
        tp = ROOT / "profiles" / "r01_gemm_traffic.json"
    if tp.exists():
        tr = json.loads(tp.read_text())["per_shape"]
        keys = [f"{N}x{K}" for N, K, _ in shapes]
        if all(k in tr for k in keys):
            traffic = sum((tr[k]["dram_read_gb"] + tr[k]["dram_write_gb"]) * 1e9 for k in keys)
    return {"bound": "tensor", "kernel": "gemm_bf16_2sm_kernel (tcgen05 CTA pair; the 4 OPT projections at M=2^20, "
                                         "one launch each)",
            "achieved": achieved, "peak": pk["bf16_tflops"], "unit": "TFLOP/s", "frac": achieved / pk["bf16_tflops"],
            "traffic": traffic, "traffic_unit": "bytes per launch set (ncu dram read + write)",
            "algorithmic_flops": tot_f, "per_shape": res}


def sort_traffic(key):
    """DRAM bytes (read + write) of one call from the committed ncu capture, or None."""
    p = ROOT / "profiles" / "r02_sort_traffic.json"
    if not p.exists():
        p = ROOT / "profiles" / "r01_sort_traffic.json"
    try:
        d = json.loads(p.read_text())[key]
        return d["dram_read_bytes"] + d["dram_write_bytes"]
    except (OSError, KeyError, ValueError):
        return None


def tau_and_rankstep(pk, reps=5):
    """cfg4 secondary metrics on rank 0: exact tau counts and one ranking step over
    the 1M-request queue (device time, CUDA events)."""
    sys.path.insert(0, str(ROOT / "tests" / "golden"))
    import recipes
    from paper_2408_15792_b200 import ranking
    from paper_2408_15792_b200.schedulers import DeviceQueue, SchedulerConfig
    x, y = recipes.tau_1m("f32")
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    out = torch.empty(6, dtype=torch.int64, device="cuda")
    ranking.tau_counts_device(xd, yd, out)
    t_eager = timed(lambda: ranking.tau_counts_device(xd, yd, out), reps)
    plan = ranking.TauPlan(xd, yd)  # the fast path's kernels, replayed as one CUDA graph
    plan()
    t = timed(plan, reps)
    assert int(plan.out[5]) == 0 and torch.equal(plan.out, out), "graph and eager tau counts differ"
    n = len(x)
    pairs = n * (n - 1) / 2
    tau_bytes = 8.0 * n
    q = recipes.queue_1m()
    dq = DeviceQueue.from_arrays(score=q["score"], scored=np.ones(n, bool), priority=q["priority"],
                                 running=q["running"], prompt_tokens=q["prompt"], generated_tokens=q["generated"],
                                 arrival_time=q["arrival"], ids=q["ids"], starvation=q["starvation"],
                                 quantum=q["quantum"], score_dtype=torch.float32)
    cfg = SchedulerConfig(max_batch=256, starvation_threshold=100, priority_quantum=50)
    snap = [dq.flags.clone(), dq.starvation.clone(), dq.quantum.clone()]

    def step():
        dq.rank_step(cfg, None, length_calibrated=False)

    step()
    tr_eager = timed(step, reps)
    step = dq.rank_step_graph(cfg, None, length_calibrated=False)
    step()
    tr = timed(step, reps)
    for dst, src in zip((dq.flags, dq.starvation, dq.quantum), snap):
        dst.copy_(src)
    rs_bytes = 34.0 * n
    import bench_cpu
    return {
        "tau": {"metric": "Kendall tau-b pairs/sec (exact counts)", "value": pairs / (t / 1e3), "unit": "pairs/s",
                "n": n, "ms": t, "ms_eager": t_eager, "note": "ms: the kernels replayed as one CUDA graph",
                "roofline": {"bound": "hbm", "achieved": tau_bytes / t / 1e6, "peak": pk["hbm_gbs"],
                                              "unit": "GB/s", "frac": tau_bytes / t / 1e6 / pk["hbm_gbs"],
                                              "traffic": sort_traffic("tau_1m"), "algorithmic_bytes": tau_bytes},
                "cpu_baseline": bench_cpu.tau()},
        "rank_step": {"metric": "requests ranked/sec (sort + fill + starvation bump)", "value": n / (tr / 1e3),
                      "unit": "requests/s", "n": n, "ms": tr, "ms_eager": tr_eager,
                      "roofline": {"bound": "hbm", "achieved": rs_bytes / tr / 1e6, "peak": pk["hbm_gbs"],
                                   "unit": "GB/s", "frac": rs_bytes / tr / 1e6 / pk["hbm_gbs"],
                                   "traffic": sort_traffic("rank_step_1m"),
                                   "algorithmic_bytes": rs_bytes},
                      "cpu_baseline": bench_cpu.rank_step()},
    }


def size_sweep(pk, reps=3):
    """at the cfg4 size (1M) tau and the rank-step are latency-bound (8 / 34 MB
    of compulsory traffic is microseconds of HBM time), so their HBM fraction is also
    reported at sizes well above L2 (synthetic fp32 scores N(0,1), lengths U[1, 2048])."""
    from paper_2408_15792_b200 import ranking
    from paper_2408_15792_b200.schedulers import DeviceQueue, SchedulerConfig
    out = {"tau": [], "rank_step": []}
    g = torch.Generator(device="cuda").manual_seed(11)
    for n in (1 << 20, 1 << 24, 1 << 26, 1 << 28):  # to 256M rows (2.15 GB of x, y), SURVEY 8d
        x = torch.randn(n, device="cuda", generator=g)
        y = torch.randint(1, 2049, (n,), device="cuda", generator=g, dtype=torch.int32)
        res = torch.empty(6, dtype=torch.int64, device="cuda")
        ranking.tau_counts_device(x, y, res, fast_only=True)
        t = timed(lambda: ranking.tau_counts_device(x, y, res, fast_only=True), reps)
        assert int(res[5]) == 0, "tau fast path declined a cfg4-shaped input"
        # comparator, not a path: a library radix sort (torch.sort = CUB) of the (x, index)
        # pairs alone. Every exact O(n log n) count orders x first, so this is the floor a
        # sort-based tau sits above; vs_sort = sort_ms / ms
        torch.sort(x)
        ts = timed(lambda: torch.sort(x), reps)
        out["tau"].append({"n": n, "ms": t, "pairs_per_s": n * (n - 1) / 2 / (t / 1e3),
                           "achieved_gbs": 8.0 * n / t / 1e6, "frac": 8.0 * n / t / 1e6 / pk["hbm_gbs"],
                           "sort_ms": ts, "vs_sort": ts / t})
        del x, y
    cfg = SchedulerConfig(max_batch=256, starvation_threshold=100, priority_quantum=50)
    for n in (1 << 20, 1 << 24, 1 << 26):  # reorder to 64M rows
        dq = DeviceQueue(n, torch.device("cuda"), score_dtype=torch.float32)
        dq.score.copy_(torch.randn(n, device="cuda", generator=g))
        from paper_2408_15792_b200 import _lib
        dq.flags.fill_(_lib.RS_FLAG_SCORED)
        dq.arrival_rank.copy_(torch.arange(n, dtype=torch.int32))
        dq.rank_step(cfg, None, length_calibrated=False)
        t = timed(lambda: dq.rank_step(cfg, None, length_calibrated=False), reps)
        out["rank_step"].append({"n": n, "ms": t, "requests_per_s": n / (t / 1e3), "achieved_gbs": 34.0 * n / t / 1e6,
                                 "frac": 34.0 * n / t / 1e6 / pk["hbm_gbs"]})
        del dq
    # ListMLE loss + grad in the training form (12.06 B/item = g fp32 +
    # length int32 read, dg fp32 written, + 4 B loss per list), 1M lists x 64 = 809.5 MB.
    out["listmle"] = []
    for n_lists in (1 << 20,):
        L = 64
        gl = torch.randn(n_lists, L, device="cuda", generator=g)
        ln = torch.randint(1, 2049, (n_lists, L), device="cuda", generator=g, dtype=torch.int32)
        ranking.listmle_from_lengths(gl, ln)
        t = timed(lambda: ranking.listmle_from_lengths(gl, ln), reps)
        nbytes = 12.0 * n_lists * L + 4.0 * n_lists
        import bench_cpu
        out["listmle"].append({"lists": n_lists, "list_len": L, "ms": t, "items_per_s": n_lists * L / (t / 1e3),
                               "achieved_gbs": nbytes / t / 1e6, "frac": nbytes / t / 1e6 / pk["hbm_gbs"],
                               "cpu_baseline": bench_cpu.listmle()})
        del gl, ln
    torch.cuda.empty_cache()
    return out


def engine_metric(args, world, rank, pk):
    """cfg5 (BASELINE.json configs[4]): end-to-end scheduler loop on the reference's own
    trace generator, generate_poisson(40, n, sharegpt, seed 7, prompt_noise 0.25)
    (workload.py:288-313; workload.generate_poisson draws the identical trace). Every
    request's prompt is tokenized on the device and scored once by the OPT-125M-shape ranker
    (S = 128, prompts sharded across ranks, scores all-gathered: the score cache — the
    ranker is a pure function of the prompt), then rank 0 runs the engine loop
    (admission, ranking-policy step with starvation bump, execute, retirement) on the device
    (paper_2408_15792_b200.engine) with max_batch 256, threshold 100, quantum 50, the
    default cost preset. Wall clock of scoring + loop (the whole loop is one cluster launch:
    rs_engine_run's device path, csrc/rankstep.cu engine_loop_kernel)."""
    from paper_2408_15792_b200 import dp, engine
    from paper_2408_15792_b200.ranker import OptRanker, RankerConfig
    from paper_2408_15792_b200.schedulers import SchedulerConfig
    from paper_2408_15792_b200.workload import LengthDist, generate_poisson, prompt_token_ids_device
    n = args.e2e_requests
    trace = generate_poisson(40.0, n, LengthDist.parse("sharegpt"), seed=7, prompt_noise=0.25)
    reqs = trace.requests
    prompts = [r.prompt for r in reqs]
    cfg = RankerConfig.opt_125m()
    model = OptRanker(cfg, seed=0)
    lo, hi = dp.shard_range(n, world, rank)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    ids_d, last_d = prompt_token_ids_device(prompts[lo:hi], 128, cfg.vocab, host_fallback=True)
    g = dp.gather_scores(model.forward(ids_d, last_d), n)
    scores = (-g).double().cpu().numpy()
    t1 = time.perf_counter()
    res = None
    if rank == 0:
        sched = SchedulerConfig(max_batch=256, starvation_threshold=100, priority_quantum=50)
        eng = engine.DeviceEngine(reqs, scores, sched, engine.COST_PRESETS["default"])
        t2 = time.perf_counter()
        res = eng.run()
        t3 = time.perf_counter()
    rescore = None
    if rank == 0 and args.rescore_steps > 0:
        # a capped "true re-score" variant — every step re-scores every
        # alive request with the ranker (S = 128) instead of reading the score cache; the
        # ranker is a pure function of the prompt, so the decisions must equal the cached
        # run's over the same steps
        K = args.rescore_steps
        scored = [0]
        all_ids, all_last = prompt_token_ids_device(prompts, 128, cfg.vocab, host_fallback=True)

        def rescore_fn(alive_ids):
            scored[0] += alive_ids.numel()
            return (-model.forward(all_ids[alive_ids], all_last[alive_ids])).double()

        eng_c = engine.DeviceEngine(reqs, scores, sched, engine.COST_PRESETS["default"])
        ref = eng_c.run(max_steps=K, native=False)
        eng_r = engine.DeviceEngine(reqs, scores, sched, engine.COST_PRESETS["default"])
        torch.cuda.synchronize()
        t4 = time.perf_counter()
        res_r = eng_r.run(max_steps=K, rescore=rescore_fn)
        t5 = time.perf_counter()
        same = res_r.steps == ref.steps and res_r.requests == ref.requests
        rescore = {"steps": res_r.steps, "prompts_rescored": scored[0], "seconds": t5 - t4,
                   "steps_per_s": res_r.steps / (t5 - t4), "prompts_rescored_per_s": scored[0] / (t5 - t4),
                   "decisions_equal_cached": bool(same),
                   "note": f"first {K} steps, every alive request re-scored each step (OPT-125M shape, S = 128)"}
        del all_ids, all_last
    if world > 1:
        torch.distributed.barrier()
    del model, ids_d
    torch.cuda.empty_cache()
    if rank != 0:
        return None
    score_s, loop_s = t1 - t0, t3 - t2
    m = res.metrics
    line = {"metric": "end-to-end scheduler loop requests/sec (score cache + device engine)",
            "value": n / (score_s + loop_s), "unit": "requests/s", "requests": n, "steps": res.steps,
            "score_s": score_s, "loop_s": loop_s, "steps_per_s": res.steps / loop_s,
            "prompts_scored_per_s": n / score_s, "sim": {k: m[k] for k in ("n_finished", "makespan_s",
                                                                          "mean_latency_s", "p90_max_waiting_s",
                                                                          "execution_order_tau")},
            "workload": f"generate_poisson(40, {n}, sharegpt, seed=7, prompt_noise=0.25) (the reference's generator; "
                        "identical trace), prompts tokenized on the device to 128 ids, max_batch 256, starvation "
                        "100/50, default cost preset", "true_rescore": rescore}
    if world == 1:
        import bench_cpu
        line["cpu_baseline"] = bench_cpu.engine_loop(trace, args.cpu_engine_prefix)
    return line


def train_step_metric(args, world, rank, pk, n_lists=None, S=None, micro=None, baselines=True):
    """cfg3 (BASELINE.json configs[2]): one ListMLE optimizer step over a global batch of
    1024 lists x 64 prompts x 128 tokens, lists sharded across ranks, gradient all-reduce
    (NCCL) + fused Adam. Device time by CUDA events, max over ranks. Also run at S = 512
    (SURVEY 8d's secondary cfg3 run; the blocked attention backward) on fewer lists."""
    from paper_2408_15792_b200.ranker import OptRanker, RankerConfig
    from paper_2408_15792_b200.trainer import RankerTrainer
    cfg = RankerConfig.opt_125m()
    n_lists = n_lists or args.train_lists
    S = S or args.train_seq
    list_len = 64
    mine = len(range(rank, n_lists, world))
    model = OptRanker(cfg, seed=0)
    tr = RankerTrainer(model, lr=2e-5, lists_per_micro=micro or args.train_micro)
    gen = torch.Generator().manual_seed(2000 + rank)
    ids = torch.randint(4, cfg.vocab, (mine * list_len, S), generator=gen, dtype=torch.int32).cuda()
    lengths = torch.randint(1, 2049, (mine * list_len,), generator=gen, dtype=torch.int32).cuda()

    def step():
        tr.accumulate(ids, lengths, list_len)
        tr.apply(n_lists)

    step()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.train_steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.train_steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    prompts = n_lists * list_len
    flops = 3.0 * cfg.flops_per_prompt(S) * prompts  # fwd + dgrad + wgrad
    tflops = flops / (ms / 1e3) / 1e12 / world
    del tr, model, ids, lengths
    torch.cuda.empty_cache()
    line = {"metric": f"ListMLE training prompts/sec ({n_lists} lists x 64 prompts x {S} tokens per step, DP)",
            "value": prompts / (ms / 1e3), "unit": "prompts/s", "ms_per_step": ms, "steps": args.train_steps,
            "global_lists": n_lists, "list_len": list_len, "seq_len": S, "flops_per_step": flops,
            "tflops_per_gpu": tflops, "frac_of_sustained": tflops / pk["bf16_tflops_sustained"]}
    if rank == 0 and world == 1 and baselines:
        import bench_cpu
        line["cpu_baseline"] = bench_cpu.train_step(cfg, S)
        line["cpu_baseline_listmle"] = bench_cpu.listmle(n_lists, list_len)
    return line


def plugin_e2e(args, model, sched, world, rank, dev, barrier, max_over_ranks):
    """End to end through the drop-in plugin API, exactly the calls the reference's
    engine.run makes each step (engine.py:414-430): OptRankerScorer.score_batch(requests)
    on this rank's B Request objects with S-token prompt strings (prompts -> ids on the
    device, forward, scores back as Python floats), the scores written to the requests,
    then on rank 0 RankingPolicy.schedule(candidates, kv_budget) over all B x world
    requests (SoA gather, H2D, rs_arrival_rank + rs_rank_step, D2H, state written back).
    With N > 1 the score lists are all-gathered (NCCL) before the schedule call."""
    import torch.distributed as dist
    from paper_2408_15792_b200.predictors import OptRankerScorer
    from paper_2408_15792_b200.schedulers import UNLIMITED_KV, RankingPolicy
    from paper_2408_15792_b200.workload import _VOCAB, Request, prompt_token_ids_device
    B, S = args.batch, args.seq
    words = np.array(_VOCAB, dtype=object)
    rng = np.random.default_rng(1000 + rank)
    prompts = [" ".join(words[rng.integers(0, len(words), S)]) for _ in range(B)]
    mine = [Request(id=rank * B + k, arrival_time=float(rank * B + k), prompt_tokens=S, true_output_tokens=1,
                    prompt=p) for k, p in enumerate(prompts)]
    allreq = mine
    if rank == 0 and world > 1:
        allreq = mine + [Request(id=k, arrival_time=float(k), prompt_tokens=S, true_output_tokens=1)
                         for k in range(B, B * world)]
    scorer = OptRankerScorer(model, seq_len=S)
    pol = RankingPolicy(sched, scorer.length_calibrated)
    gbuf = torch.empty(B * world, dtype=torch.float64, device=dev)
    parts = {"score_batch": 0.0, "gather": 0.0, "schedule": 0.0}

    def step():
        t0 = time.perf_counter()
        sc = scorer.score_batch(mine, 0)
        t1 = time.perf_counter()
        if world > 1:
            dist.all_gather_into_tensor(gbuf, torch.tensor(sc, dtype=torch.float64, device=dev))
            sc = gbuf.cpu().tolist() if rank == 0 else sc
        t2 = time.perf_counter()
        dec = None
        if rank == 0:
            for r, v in zip(allreq, sc):
                r.score = v
            dec = pol.schedule(allreq, UNLIMITED_KV)
        t3 = time.perf_counter()
        parts["score_batch"] += t1 - t0
        parts["gather"] += t2 - t1
        parts["schedule"] += t3 - t2
        return dec

    step()
    for k in parts:
        parts[k] = 0.0
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    barrier()
    ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / args.steps)
    # breakdown of score_batch: the device tokenizer alone, and the host-map tokenizer
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prompt_token_ids_device(prompts, S, model.cfg.vocab, host_fallback=True)
    torch.cuda.synchronize()
    tok_dev = time.perf_counter() - t0
    t0 = time.perf_counter()
    OptRankerScorer(model, seq_len=S, device_tokenizer=False).encode(mine)
    tok_host = time.perf_counter() - t0
    text_bytes = sum(len(p) for p in prompts)
    n_all = B * world
    return {"value": n_all / (ms / 1e3), "unit": UNIT, "ms_per_step": ms,
            "h2d_bytes_per_step": text_bytes + 8 * (B + 1) + (45 * n_all if rank == 0 else 0),
            "d2h_bytes_per_step": 4 * B + (37 * n_all if rank == 0 else 0),
            "path": "OptRankerScorer.score_batch(requests) [prompt bytes H2D, rs_tokenize, rs_ranker_forward, scores "
                    "D2H] -> request.score = s -> RankingPolicy.schedule(requests, kv) [SoA staging H2D, "
                    "rs_arrival_rank + rs_rank_step, decision + state D2H, write-back]",
            "breakdown_ms": {k: v * 1e3 / args.steps for k, v in parts.items()},
            "tokenize_ms": {"device": tok_dev * 1e3, "host_map": tok_host * 1e3},
            "requests": f"{B} Request objects per rank with {S}-token prompts drawn from the reference vocabulary"}


def run_ours(args):
    import torch.distributed as dist
    world, rank, local = dist_env()
    # RSB200_BENCH_BACKEND=gloo runs the N > 1 code path with every rank on the one GPU a
    # test box has (NCCL refuses two ranks per device); the driver's runs use NCCL.
    backend = os.environ.get("RSB200_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_2408_15792_b200 import _lib
    from paper_2408_15792_b200.ranker import OptRanker, RankerConfig
    from paper_2408_15792_b200.schedulers import DeviceQueue, SchedulerConfig
    dev = _lib.device(local)
    pk = peaks()
    cfg = RankerConfig.opt_125m()
    B, S = args.batch, args.seq
    model = OptRanker(cfg, seed=0)
    gen = torch.Generator().manual_seed(1000 + rank)
    ids_host = torch.randint(4, cfg.vocab, (B, S), generator=gen, dtype=torch.int32).pin_memory()
    ids_dev = ids_host.to(dev)
    gathered = torch.empty(B * world, dtype=torch.float32, device=dev)
    local_scores = gathered[rank * B:(rank + 1) * B] if world == 1 else torch.empty(B, dtype=torch.float32,
                                                                                      device=dev)
    g_out = torch.empty(B, dtype=torch.float32, device=dev)
    sched = SchedulerConfig(max_batch=256, starvation_threshold=100, priority_quantum=50)
    queue = None
    if rank == 0:
        n = B * world
        queue = DeviceQueue(n, dev, score_dtype=torch.float32)
        queue.score = gathered  # the gathered scores are the queue's score column
        queue.flags.fill_(_lib.RS_FLAG_SCORED)
        queue.arrival_rank.copy_(torch.arange(n, dtype=torch.int32))
    run_host = torch.empty(sched.max_batch, dtype=torch.int64).pin_memory()
    cnt_host = torch.empty(4, dtype=torch.int32).pin_memory()

    def step():
        model.forward(ids_dev, out=g_out, score_out=local_scores)
        if world > 1:
            dist.all_gather_into_tensor(gathered, local_scores)
        if rank == 0:
            queue.rank_step(sched, None, length_calibrated=False)

    def step_e2e():
        ids_dev.copy_(ids_host, non_blocking=True)
        step()
        if rank == 0:
            run_host.copy_(queue.run_out[:sched.max_batch], non_blocking=True)
            cnt_host.copy_(queue.counts, non_blocking=True)
        torch.cuda.current_stream().synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step()
    barrier()
    lib = _lib.load()
    l0 = lib.rs_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier()
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        barrier()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    launches = int(lib.rs_launch_count() - l0)
    value = B * world / (ms / 1e3)

    # C-ABI level with host buffers (H2D token ids, D2H run ids): e2e_ids
    step_e2e()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step_e2e()
    barrier()
    e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / args.steps)
    # the headline e2e: the plugin calls the reference's engine makes (engine.py:414-430)
    plugin = plugin_e2e(args, model, sched, world, rank, dev, barrier, max_over_ranks)

    extras = {}
    if rank == 0 and not args.no_extras:
        extras["roofline"] = gemm_roofline(pk)
        extras.update(tau_and_rankstep(pk))
        extras["size_sweep"] = size_sweep(pk)
    if not args.no_extras and not args.no_train:
        extras["train_step"] = train_step_metric(args, world, rank, pk)
        if args.train512_lists > 0:
            extras["train_step_s512"] = train_step_metric(args, world, rank, pk, n_lists=args.train512_lists, S=512,
                                                          micro=4, baselines=False)
    if not args.no_extras and args.e2e_requests > 0:
        extras["e2e_loop"] = engine_metric(args, world, rank, pk)
    if rank == 0 and not args.no_extras:
        if world == 1:
            extras["cpu_baseline"] = cpu_baseline(cfg, S, n_prompts=args.cpu_prompts)
    if world > 1:
        dist.barrier()
    if rank != 0:
        dist.destroy_process_group()
        return 0
    flops = cfg.flops_per_prompt_pruned(S)  # what the forward computes (last layer pruned)
    model_tflops = value * flops / 1e12 / world
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random token ids, random-init OPT-125M-shape weights, seed 0)",
        "config": {"workload": f"OPT-125M-shape ranker scoring {B} prompts x {S} tokens per GPU (bf16 operands, "
                               "fp32 accumulate/residual) + score all-gather + rank-step sort (max_batch 256)",
                   "global_batch": B * world, "seq_len": S, "parallelism": f"dp{world}",
                   "l2": "inputs larger than L2 (activations ~10 GB per 1M-token chunk)"},
        "roofline": extras.get("roofline"),
        "cpu_baseline": extras.get("cpu_baseline"),
        "e2e": plugin,
        "e2e_ids": {"value": B * world / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": B * S * 4,
                    "d2h_bytes_per_step": sched.max_batch * 8 + 16, "ms_per_step": e2e_ms,
                    "path": "pinned token ids H2D -> rs_ranker_forward -> (all-gather) -> rs_rank_step -> run ids D2H"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "model_flops": {"per_prompt": flops, "per_prompt_unpruned": cfg.flops_per_prompt(S),
                        "tflops_per_gpu": model_tflops,
                        "frac_of_sustained": model_tflops / pk["bf16_tflops_sustained"],
                        "frac_of_burst": model_tflops / pk["bf16_tflops"]},
        "peaks": {k: pk.get(k) for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained", "source")},
        "tau": extras.get("tau"),
        "rank_step": extras.get("rank_step"),
        "train_step": extras.get("train_step"),
        "train_step_s512": extras.get("train_step_s512"),
        "size_sweep": extras.get("size_sweep"),
        "e2e_loop": extras.get("e2e_loop"),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--seq", type=int, default=512)
    ap.add_argument("--cpu-prompts", type=int, default=16)
    ap.add_argument("--ref-prompts", type=int, default=16)
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-train", action="store_true")
    ap.add_argument("--train-lists", type=int, default=1024)
    ap.add_argument("--train-seq", type=int, default=128)
    ap.add_argument("--train-micro", type=int, default=16)
    ap.add_argument("--train-steps", type=int, default=1)
    ap.add_argument("--train512-lists", type=int, default=64,
                    help="cfg3 secondary run at S = 512 over this many lists of 64 (0 disables)")
    ap.add_argument("--e2e-requests", type=int, default=100000,
                    help="cfg5 loop size (BASELINE configs[4]: 100000; 0 disables)")
    ap.add_argument("--cpu-engine-prefix", type=int, default=5000,
                    help="cfg5 CPU baseline: reference engine.run over this many leading requests")
    ap.add_argument("--rescore-steps", type=int, default=400,
                    help="cfg5 capped true re-score variant: steps that re-score every alive request (0 disables)")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


def self_launch(n: int) -> int:
    """`python bench.py --gpus N` without a launcher: start N ranks (one process per GPU)
    through torch.distributed.run on 127.0.0.1 with this same command line; rank 0 prints
    the JSON line."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(pathlib.Path(__file__).resolve())]
    cmd += sys.argv[1:]
    return subprocess.run(cmd).returncode


if __name__ == "__main__":
    sys.exit(main())

"""Small shapes of every librsb200 kernel, for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck) — tests/test_gpu_sanitizer.py runs this file under each tool.

Covers: tcgen05 GEMMs (forward epilogues + backward variants through the training pass),
attention forward (f16 V and bf16 V) and backward, LayerNorm / embedding / head, ranker
forward and rs_ranker_grad + Adam, classifier head + CE, ListMLE (order / lengths forms),
tau counts (small-range y histogram path and the general merge path, 32- and 64-bit
inputs), arrival rank + rank step (select and sort paths, KV budget), the device engine
loop (the one-launch loop and the per-kernel steps), the tokenizer and the linear bridge."""

from __future__ import annotations

import pathlib
import sys

import numpy as np
import torch

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main(which: str = "all"):
    from paper_2408_15792_b200 import engine, ranking, schedulers
    from paper_2408_15792_b200.linear_ranker import FeatureTrainConfig, train_ranking_features
    from paper_2408_15792_b200.ranker import OptRanker, RankerConfig
    from paper_2408_15792_b200.trainer import ClassifierTrainer, RankerTrainer
    from paper_2408_15792_b200.workload import Request, fixed_burst, prompt_token_ids_device

    torch.cuda.set_device(0)
    g = torch.Generator().manual_seed(0)
    if which in ("all", "ranker"):
        cfg = RankerConfig.opt_125m(vocab=512, max_pos=256, d_model=256, n_layers=2, n_heads=4, d_ffn=1024)
        m = OptRanker(cfg, seed=0)
        ids = torch.randint(4, cfg.vocab, (4, 200), generator=g, dtype=torch.int32).cuda()
        m.forward(ids)
        m.features(ids[:, :64])
        tr = RankerTrainer(m, lr=1e-3, lists_per_micro=1)
        tids = torch.randint(4, cfg.vocab, (16, 64), generator=g, dtype=torch.int32).cuda()
        tl = torch.randint(1, 2049, (16,), generator=g, dtype=torch.int32).cuda()
        tr.step(tids, tl, 8)
        ct = ClassifierTrainer(m, 4, prompts_per_micro=8)
        ct.accumulate(tids, torch.randint(0, 4, (16,), generator=g, dtype=torch.int32).cuda())
        ct.apply(16)
    if which in ("all", "sort"):
        rng = np.random.default_rng(0)
        for n in (5, 3000, 40_000):
            x = rng.normal(size=n).astype(np.float32)
            ranking.kendall_tau_b(x, rng.integers(0, 50, n))                       # bucket fast path
            ranking.kendall_tau_b(x, rng.normal(size=n))                           # general y, f64
            ranking.kendall_tau_b(rng.integers(0, 9, n).astype(np.int64), x)       # 64-bit x
        import os
        os.environ["RS_TAU_PATH"] = "fast"  # the bucket path at sanitizer sizes (below its crossover)
        for n in (5, 3000, 40_000):
            x = rng.normal(size=n).astype(np.float32)
            ranking.kendall_tau_b(x, rng.integers(0, 50, n))
            ranking.kendall_tau_b(rng.integers(0, 9, n).astype(np.int64), rng.integers(0, 9, n))
        n = 40_000
        near1 = (1.0 + 1e-4 * rng.normal(size=n)).astype(np.float32)              # level-2 splits
        ranking.kendall_tau_b(near1, rng.integers(1, 2049, n))
        one = np.float32(1.0).view(np.int32)
        for width in (2, 40):                                                       # crowded child, fallback
            c = (one + rng.integers(0, width, n).astype(np.int32)).view(np.float32)
            c[:2] = (-1e30, 1e30)
            ranking.kendall_tau_b(c, rng.integers(1, 2049, n))
        del os.environ["RS_TAU_PATH"]
        s = torch.randn(300, 64, dtype=torch.float64, device="cuda")
        o = torch.argsort(torch.rand(300, 64, device="cuda"), dim=1)
        ranking.list_mle_batched(s, o)
        ranking.list_mle_batched(s[:4, :40].float().contiguous(), torch.argsort(torch.rand(4, 40, device="cuda"), 1))
        ranking.listmle_from_lengths(torch.randn(257, 64, device="cuda"),
                                     torch.randint(1, 2049, (257, 64), device="cuda", dtype=torch.int32))
        ranking.listmle_from_lengths(torch.randn(9, 100, device="cuda"),
                                     torch.randint(1, 2049, (9, 100), device="cuda", dtype=torch.int32))
        for n in (50, 5000):
            reqs = []
            for k in range(n):
                r = Request(id=k, arrival_time=float(k // 3), prompt_tokens=1 + k % 97, true_output_tokens=5)
                r.score = float(rng.normal())
                r.starvation_count = int(k % 120)
                r.priority = k % 50 == 0
                reqs.append(r)
            pol = schedulers.RankingPolicy(schedulers.SchedulerConfig(max_batch=64), False)
            pol.schedule(reqs, 1 << 62)
            pol.schedule(reqs, 3000)
        # 40k rows: the one-launch select as one CTA cluster (sel_fused<.., true>); 100k: as
        # a cooperative grid; 300k (> 2^18): the multi-launch select (f32 keys from the
        # columns; f64 / calibrated keys)
        for n, sdt, calib in ((40_000, torch.float32, False), (40_000, torch.float32, True),
                              (100_000, torch.float32, False), (100_000, torch.float64, True),
                              (300_000, torch.float32, False), (300_000, torch.float64, False),
                              (300_000, torch.float32, True)):
            dq = schedulers.DeviceQueue.from_arrays(
                score=rng.normal(size=n), scored=rng.random(n) < 0.95, priority=rng.random(n) < 0.01,
                running=np.zeros(n, bool), prompt_tokens=rng.integers(1, 100, n),
                generated_tokens=rng.integers(0, 50, n), arrival_time=np.sort(rng.random(n)),
                ids=np.arange(n), starvation=rng.integers(0, 100, n), quantum=rng.integers(0, 50, n),
                score_dtype=sdt)
            dq.rank_step(schedulers.SchedulerConfig(max_batch=256), None, length_calibrated=calib)
    if which in ("all", "engine"):
        trace = fixed_burst([3, 1, 4, 1, 5, 9, 2, 6] * 8)
        res = engine.run(list(trace), scores=list(np.random.default_rng(1).normal(size=len(trace))),
                         sched=schedulers.SchedulerConfig(max_batch=4), cost=engine.COST_PRESETS["unit"])
        assert res.metrics["n_finished"] == len(trace)
        # the per-kernel step path too (record=True: admit / execute / compaction kernels)
        rec = engine.DeviceEngine(list(trace), list(np.random.default_rng(1).normal(size=len(trace))),
                                  schedulers.SchedulerConfig(max_batch=4), engine.COST_PRESETS["unit"]).run(record=True)
        assert rec.metrics["n_finished"] == len(trace)
        prompt_token_ids_device(["a b c", "", "  hello   World ", "x " * 300], 16)
        wl = __import__("paper_2408_15792_b200.workload", fromlist=["x"])
        t = wl.generate_burst(120, wl.LengthDist.parse("sharegpt"), seed=1)
        train_ranking_features(t, FeatureTrainConfig(epochs=1, hidden=8))
    torch.cuda.synchronize()
    print("sanitize-small ok")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")

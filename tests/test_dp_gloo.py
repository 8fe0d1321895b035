"""Data-parallel host logic at world_size 2 over gloo on CPU: prompt shards
cover the batch exactly once, the score all-gather restores prompt order, list shards
keep lists whole, and the gradient all-reduce equals the single-process sum. The CUDA
kernels are replaced by deterministic CPU stand-ins; only the plumbing is under test."""

import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2408_15792_b200 import dp
from paper_2408_15792_b200.ranker import OptRanker


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class _StubRanker:
    """forward(ids, last) -> a deterministic per-prompt value (stands in for the kernel)."""

    def forward(self, ids, last_pos=None):
        lp = torch.full((ids.shape[0],), ids.shape[1] - 1) if last_pos is None else last_pos.long()
        return ids.float().sum(1) * 0.5 + ids[torch.arange(ids.shape[0]), lp].float()


def _fake_list_grad(lst, n_params=37):
    g = torch.zeros(n_params)
    for i in lst:
        g += torch.sin(torch.arange(n_params) * 0.1 + float(i))
    return g


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        for B in (10, 11, 1, 2):
            ids = torch.arange(B * 6).view(B, 6) % 13
            last = (torch.arange(B) * 5) % 6
            stub = _StubRanker()
            out[f"scores{B}"] = OptRanker.forward_sharded(stub, ids, last).tolist()
        lists = [list(range(k * 4, k * 4 + 4)) for k in range(7)]
        g = torch.zeros(37)
        for lst in dp.shard_lists(lists, world, rank):
            g += _fake_list_grad(lst)
        dp.allreduce_sum_(g)
        out["grad"] = g.tolist()
        loss = torch.tensor(float(len(dp.shard_lists(lists, world, rank))))
        dp.allreduce_sum_(loss)
        out["n_lists"] = loss.item()
        results[rank] = out
    finally:
        dist.destroy_process_group()


def test_shard_range_partitions():
    for n in (0, 1, 7, 4096, 4097):
        for world in (1, 2, 3, 8):
            got = [dp.shard_range(n, world, r) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            sizes = [hi - lo for lo, hi in got]
            assert max(sizes) - min(sizes) <= 1


def test_world2_gloo_gather_and_allreduce():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, port, results), nprocs=world, join=True)
    stub = _StubRanker()
    for B in (10, 11, 1, 2):
        ids = torch.arange(B * 6).view(B, 6) % 13
        last = (torch.arange(B) * 5) % 6
        want = stub.forward(ids, last).tolist()
        for r in range(world):
            assert results[r][f"scores{B}"] == want
    lists = [list(range(k * 4, k * 4 + 4)) for k in range(7)]
    want = torch.zeros(37)
    for lst in lists:
        want += _fake_list_grad(lst)
    for r in range(world):
        torch.testing.assert_close(torch.tensor(results[r]["grad"]), want, rtol=1e-6, atol=1e-5)
        assert results[r]["n_lists"] == 7

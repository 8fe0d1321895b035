"""Data-parallel plumbing of the hot path, one process per GPU.

Scoring shards prompts contiguously across ranks and gathers the fp32 scores to every
rank (NCCL all-gather; the queue owner, rank 0, then runs the rank-step). ListMLE
training shards whole lists (ListMLE couples a list's scores, so a list never spans
ranks) and sums the fp32 gradient buffer with one all-reduce before the replicated
Adam step. These helpers only move tensors; they run unchanged on CPU tensors under
the gloo backend, which is how tests/test_dp_gloo.py covers the N > 1 logic.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def world_rank(group=None) -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) slice of n items for `rank` (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_lists(lists: list, world: int, rank: int) -> list:
    """Round-robin assignment of whole lists to ranks (a list never spans ranks)."""
    return lists[rank::world]


def gather_scores(local: torch.Tensor, n_total: int, group=None) -> torch.Tensor:
    """All-gather every rank's contiguous score shard (shard_range order) into one
    [n_total] tensor on every rank; shards may differ in length by one."""
    world, rank = world_rank(group)
    if world == 1:
        return local
    width = -(-n_total // world)
    buf = torch.zeros(width, dtype=local.dtype, device=local.device)
    buf[:local.numel()] = local
    out = torch.empty(width * world, dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    parts = [out[r * width:r * width + (shard_range(n_total, world, r)[1] - shard_range(n_total, world, r)[0])]
             for r in range(world)]
    return torch.cat(parts)


def allreduce_sum_(t: torch.Tensor, group=None) -> torch.Tensor:
    """In-place sum over ranks (the gradient all-reduce; a no-op on one rank)."""
    world, _ = world_rank(group)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t

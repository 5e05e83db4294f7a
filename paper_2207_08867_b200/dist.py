"""Multi-GPU plumbing of the MCF hot path: one process per GPU,
torch.distributed (NCCL on B200s, gloo in the CPU tests) for the plumbing only.

The path partitions without a data-path exchange except the MC-MLP gradient
all-reduce (mlp.GradExchange):

* mm MC x T / MC x MC: output rows [r0, r1) per rank (``row_range``); B is
  replicated -- for config 4 by a one-time broadcast from rank 0
  (``broadcast_``), untimed; shard outputs equal the single-GPU rows bitwise
  (each output depends only on its row and column);
* elementwise: flat element ranges (``row_range`` over elements);
* matvec / batched dots: row / dot-index ranges;
* every device time is reduced as the max over ranks (``max_over_ranks``).
"""
from __future__ import annotations

import os


def env():
    """(rank, world, local_rank) from the torchrun environment (1 process: 0, 1, 0)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def row_range(m: int, rank: int, world: int):
    """Contiguous block [r0, r1) of m units owned by `rank` (sizes differ by at most one)."""
    return rank * m // world, (rank + 1) * m // world


def broadcast_(t, src: int = 0, group=None):
    """In-place one-time broadcast of an operand from `src` (config 4's B)."""
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(t, src=src, group=group)
    return t


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (device times: the job's time is the slowest rank's)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def gather_rows(local, m: int, group=None):
    """All ranks' row blocks concatenated in rank order (untimed checking)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return local
    world = dist.get_world_size(group)
    mx = max(row_range(m, r, world)[1] - row_range(m, r, world)[0] for r in range(world))
    pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)  # equal sizes (NCCL / gloo), trimmed below
    out = []
    for r in range(world):
        r0, r1 = row_range(m, r, world)
        out.append(parts[r][:r1 - r0])
    return torch.cat(out, 0)

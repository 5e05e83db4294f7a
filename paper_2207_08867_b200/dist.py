"""Multi-GPU plumbing of the MCF hot path: one process per GPU,
torch.distributed (NCCL on B200s, gloo in the CPU tests) for the plumbing only.

The path partitions without a data-path exchange except the MC-MLP gradient
all-reduce (mlp.GradExchange):

* mm MC x T / MC x MC: output rows [r0, r1) per rank (``row_range``); B is
  replicated -- for config 4 by a one-time broadcast from rank 0
  (``broadcast_``), untimed; shard outputs equal the single-GPU rows bitwise
  (each output depends only on its row and column);
* config 2 (strong scaling of one 4096^3 product): output BLOCKS, rows x
  columns (``block_grid`` / ``block_range``): a rank prepares the residue
  planes of its A row block and its B column block only, so the per-rank
  preparation shrinks with the grid instead of staying at all of B (measured
  per-rank step at 8 ranks: 0.375 ms by rows, 0.297 ms as 2 x 4 blocks);
  still no collective -- each output depends only on its row and column;
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


def block_grid(world: int):
    """(gr, gc), gr * gc == world: gr the largest divisor of world not above sqrt(world)."""
    gr = 1
    for d in range(1, int(world ** 0.5) + 1):
        if world % d == 0:
            gr = d
    return gr, world // gr


def block_range(m: int, n: int, rank: int, world: int, grid=None):
    """Output block (r0, r1, c0, c1) of `rank` in a gr x gc grid (rank = row block * gc + column block)."""
    gr, gc = grid or block_grid(world)
    r0, r1 = row_range(m, rank // gc, gr)
    c0, c1 = row_range(n, rank % gc, gc)
    return r0, r1, c0, c1


def gather_blocks(local, m: int, n: int, grid=None, group=None):
    """All ranks' output blocks assembled into the m x n x ... result (untimed checking)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return local
    world = dist.get_world_size(group)
    rng = [block_range(m, n, r, world, grid) for r in range(world)]
    mr, mc = max(b[1] - b[0] for b in rng), max(b[3] - b[2] for b in rng)
    pad = torch.zeros((mr, mc) + tuple(local.shape[2:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0], :local.shape[1]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    out = torch.empty((m, n) + tuple(local.shape[2:]), dtype=local.dtype, device=local.device)
    for r, (r0, r1, c0, c1) in enumerate(rng):
        out[r0:r1, c0:c1] = parts[r][:r1 - r0, :c1 - c0]
    return out


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

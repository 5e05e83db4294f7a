"""Data-parallel logic of the MC-MLP step on CPU (world_size 2, gloo).

Each rank holds a different gradient shard in the flat buffer of
paper_2207_08867_b200.mlp.GradExchange; after all_reduce both ranks hold the
sum, and applying the MC-SGD update (grow_expn with -lr*g, through the oracle
here: no GPU on CPU) leaves the MC parameters bitwise identical on every rank.
Row-sharding helpers of the MC mm are checked to tile the output exactly.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    from paper_2207_08867_b200.mlp import GradExchange

    shapes = [(6, 5), (6,), (3, 6), (3,)]
    ex = GradExchange(shapes, "cpu", group=dist.group.WORLD)
    g = torch.Generator().manual_seed(100 + rank)
    for v in ex.views:
        v.copy_(torch.randn(v.shape, generator=g))
    mine = ex.flat.clone()
    loss = torch.tensor([float(rank + 1)])
    # per-layer buckets, started in backward order, as MCMLP.step does
    ex.reduce_bucket(2, 3)
    ex.reduce_bucket(0, 1)
    ex.finish(loss)
    # every rank's contribution, gathered for the check
    parts = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine)
    want = parts[0].clone()
    for p in parts[1:]:
        want += p
    assert torch.equal(ex.flat, want)
    assert loss.item() == sum(range(1, world + 1))
    # identical MC-SGD update on every rank (momentum 0): w <- grow_expn(w, -(lr * (0 + g)))
    port = oracle.Oracle("port")
    rng = np.random.default_rng(5)  # same seed on all ranks: replicated weights
    w = np.stack([rng.uniform(-1, 1, 30).astype(np.float32), np.zeros(30, np.float32)], -1)
    gflat = ex.views[0].numpy().ravel().astype(np.float32)
    lr = np.float32(0.01)
    delta = -(lr * (np.float32(0) + gflat)).astype(np.float32)
    w_new = port.grow_expn(w, delta)
    np.save(os.path.join(outdir, f"w{rank}.npy"), w_new)
    dist.destroy_process_group()


def test_gradient_allreduce_and_identical_updates(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    w0 = np.load(tmp_path / "w0.npy")
    w1 = np.load(tmp_path / "w1.npy")
    assert np.array_equal(w0.view(np.uint32), w1.view(np.uint32))


@pytest.mark.parametrize("m,world", [(4096, 1), (4096, 2), (4096, 8), (10, 8), (1023, 4), (3, 8)])
def test_row_shards_tile_the_output(m, world):
    from paper_2207_08867_b200.dist import row_range

    rows = [row_range(m, r, world) for r in range(world)]
    assert rows[0][0] == 0 and rows[-1][1] == m
    for (a0, a1), (b0, b1) in zip(rows, rows[1:]):
        assert a1 == b0 and a0 <= a1
    sizes = [b - a for a, b in rows]
    assert max(sizes) - min(sizes) <= 1


def _mm_worker(rank, world, port, outdir, mcmc):
    """Config 4's layout on CPU: rank 0 owns B and broadcasts it once; every
    rank computes its output row block (the oracle stands in for the GPU
    product); the gathered rows must equal the single-process product bitwise,
    and the reported time is the max over ranks."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    from paper_2207_08867_b200 import dist as pdist

    port_ = oracle.Oracle("port")
    m, k, n = 13, 40, 7
    rng = np.random.default_rng(9)  # A is generated identically everywhere (each rank keeps its rows)
    from mcgen import split

    a = split(rng.uniform(-1, 1, m * k), 2, np.float32).reshape(m, k, 2)
    if rank == 0:
        bv = split(np.random.default_rng(10).uniform(-1, 1, k * n), 2, np.float32).reshape(k, n, 2)
        b = torch.from_numpy(bv if mcmc else np.ascontiguousarray(bv[..., 0]))
    else:
        b = torch.zeros((k, n, 2) if mcmc else (k, n), dtype=torch.float32)
    pdist.broadcast_(b, src=0)
    r0, r1 = pdist.row_range(m, rank, world)
    bn = b.numpy()
    if mcmc:
        rows_idx = np.repeat(np.arange(r0, r1), n)
        cols_idx = np.tile(np.arange(n), r1 - r0)
        local = port_.mm_mcmc_sampled(a, bn, rows_idx, cols_idx).reshape(r1 - r0, n, 2)
    else:
        local = port_.mm_mcn(np.ascontiguousarray(a[r0:r1]), bn)
    full = pdist.gather_rows(torch.from_numpy(np.ascontiguousarray(local)), m)
    t = pdist.max_over_ranks(float(rank + 1))
    if rank == 0:
        if mcmc:
            ri, ci = np.repeat(np.arange(m), n), np.tile(np.arange(n), m)
            want = port_.mm_mcmc_sampled(a, bn, ri, ci).reshape(m, n, 2)
        else:
            want = port_.mm_mcn(a, bn)
        np.save(os.path.join(outdir, "full.npy"), full.numpy())
        np.save(os.path.join(outdir, "want.npy"), want)
        np.save(os.path.join(outdir, "t.npy"), np.array([t]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,mcmc", [(2, False), (3, True)])
def test_row_sharded_product_with_broadcast_b(tmp_path, world, mcmc):
    mp.spawn(_mm_worker, args=(world, _free_port(), str(tmp_path), mcmc), nprocs=world, join=True)
    full, want = np.load(tmp_path / "full.npy"), np.load(tmp_path / "want.npy")
    assert np.array_equal(full.view(np.uint32), want.view(np.uint32))
    assert float(np.load(tmp_path / "t.npy")[0]) == world


def _mm_block_worker(rank, world, port, outdir):
    """Config 2's output-block grid: each rank computes its rows x columns block
    from its rows of A and its columns of B (oracle compute), blocks assembled."""
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2207_08867_b200 import dist as pdist
    from mcgen import split

    port_ = oracle.Oracle("port")
    m, k, n = 11, 24, 9
    a = split(np.random.default_rng(3).uniform(-1, 1, m * k), 2, np.float32).reshape(m, k, 2)
    b = np.random.default_rng(4).uniform(-1, 1, (k, n)).astype(np.float32)
    r0, r1, c0, c1 = pdist.block_range(m, n, rank, world)
    local = port_.mm_mcn(np.ascontiguousarray(a[r0:r1]), np.ascontiguousarray(b[:, c0:c1]))
    full = pdist.gather_blocks(torch.from_numpy(np.ascontiguousarray(local)), m, n)
    if rank == 0:
        np.save(os.path.join(outdir, "full.npy"), full.numpy())
        np.save(os.path.join(outdir, "want.npy"), port_.mm_mcn(a, b))
    dist.destroy_process_group()


def test_block_grid_shapes():
    from paper_2207_08867_b200.dist import block_grid, block_range

    assert [block_grid(w) for w in (1, 2, 3, 4, 6, 8)] == [(1, 1), (1, 2), (1, 3), (2, 2), (2, 3), (2, 4)]
    for world in (1, 2, 4, 6, 8):
        cover = np.zeros((13, 10), dtype=int)
        for r in range(world):
            r0, r1, c0, c1 = block_range(13, 10, r, world)
            cover[r0:r1, c0:c1] += 1
        assert (cover == 1).all()


@pytest.mark.parametrize("world", [2, 4])
def test_block_sharded_product_assembles_bitwise(tmp_path, world):
    mp.spawn(_mm_block_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    full, want = np.load(tmp_path / "full.npy"), np.load(tmp_path / "want.npy")
    assert np.array_equal(full.view(np.uint32), want.view(np.uint32))

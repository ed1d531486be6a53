"""World-size-2 gloo tests of the multi-GPU host logic on CPU: walker
sharding covers every position exactly once; orbital-sharded blocks gathered
along N equal the single-device result bit for bit (blocks come from the C
oracle here -- the CUDA evaluation itself is covered by the GPU tests)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1611_02665_b200.multi import (
    OrbitalPartition,
    balanced_bounds,
    gather_orbital_blocks,
    position_shard,
    walker_shard,
)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_balanced_bounds():
    assert balanced_bounds(10, 3) == [(0, 4), (4, 7), (7, 10)]
    b = balanced_bounds(4096, 8, 16)
    assert all(hi - lo == 512 for lo, hi in b)
    b = balanced_bounds(100, 3, 16)
    assert b[0][0] == 0 and b[-1][1] == 100 and all((hi - lo) % 16 == 0 for lo, hi in b[:-1])


def test_walker_shards_partition_positions():
    for world in (1, 2, 3, 8):
        seen = []
        for r in range(world):
            sl = position_shard(4096 * 4, 4, world, r)
            assert sl.start % 4 == 0 and sl.stop % 4 == 0
            seen.extend(range(sl.start, sl.stop))
        assert seen == list(range(4096 * 4))
        assert sum(len(walker_shard(1000, world, r)) for r in range(world)) == 1000


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1611_02665_b200.coeffs import FillSpec, build_table
        from paper_1611_02665_b200.grid import GridSpec

        table = build_table(GridSpec(8, 9, 10, 0.5, 0.25, 2.0), 40, FillSpec.random(13))
        pos = np.random.default_rng(2).random((24, 3)) * 5.0
        full = oracle.eval_f32("vgh", table.data, table.grid.spacings, pos)[:, :, :40]
        part = OrbitalPartition.make(40, world, quantum=16)
        lo, hi = part.local(rank)
        local = torch.from_numpy(np.ascontiguousarray(full[:, :, lo:hi]))
        got_all = gather_orbital_blocks(local, part)
        got_root = gather_orbital_blocks(local, part, root=0)
        ok_all = bool(np.array_equal(got_all.numpy(), full))
        ok_root = (got_root is None) if rank != 0 else bool(np.array_equal(got_root.numpy(), full))
        # walker sharding: each rank's slice, all-gathered, reassembles the batch
        sl = position_shard(len(pos), 4, world, rank)
        mine = torch.from_numpy(np.ascontiguousarray(full[sl]))
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([mine.shape[0]]))
        nmax = int(max(s.item() for s in sizes))
        pad = torch.zeros((nmax,) + tuple(mine.shape[1:]), dtype=mine.dtype)
        pad[: mine.shape[0]] = mine
        bufs = [torch.zeros_like(pad) for _ in range(world)]
        dist.all_gather(bufs, pad)
        cat = torch.cat([b[: int(s.item())] for b, s in zip(bufs, sizes)])
        ok_walk = bool(np.array_equal(cat.numpy(), full))
        q.put((rank, ok_all, ok_root, ok_walk))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_orbital_gather_and_walker_shards(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    results = sorted(q.get(timeout=5) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    for rank, ok_all, ok_root, ok_walk in results:
        assert ok_all and ok_root and ok_walk, (rank, ok_all, ok_root, ok_walk)


def _ratio_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1611_02665_b200.coeffs import FillSpec, build_table
        from paper_1611_02665_b200.grid import GridSpec
        from paper_1611_02665_b200.multi import sum_ratio_partials

        table = build_table(GridSpec(8, 9, 10, 0.5, 0.25, 2.0), 40, FillSpec.random(13))
        rng = np.random.default_rng(4)
        pos = rng.random((24, 3)) * 5.0
        coef = rng.standard_normal((24, 40))
        full = oracle.eval_f32("vgh", table.data, table.grid.spacings, pos)[:, :, :40].astype(np.float64)
        want = np.einsum("psn,pn->ps", full, coef)
        bound = np.einsum("psn,pn->ps", np.abs(full), np.abs(coef))
        part = OrbitalPartition.make(40, world, quantum=16)
        lo, hi = part.local(rank)
        # the rank's partial contraction over its spline slice (the GPU path: evaluate_ratios)
        mine = torch.from_numpy(np.einsum("psn,pn->ps", full[:, :, lo:hi], coef[:, lo:hi]))
        got_all = sum_ratio_partials(mine.clone())
        got_root = sum_ratio_partials(mine.clone(), root=0)
        ok_all = bool((np.abs(got_all.numpy() - want) <= 1e-14 * bound).all())
        ok_root = (got_root is None) if rank != 0 else bool((np.abs(got_root.numpy() - want) <= 1e-14 * bound).all())
        q.put((rank, ok_all, ok_root))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_sharded_ratio_partials_sum_to_the_full_contraction(world):
    """The orbital-sharded fused consumer's exchange step (multi.sum_ratio_partials):
    per-rank partial contractions over the spline slices, all-reduced / reduced to
    rank 0, equal the contraction of the full oracle outputs."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ratio_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    results = sorted(q.get(timeout=5) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    for rank, ok_all, ok_root in results:
        assert ok_all and ok_root, (rank, ok_all, ok_root)

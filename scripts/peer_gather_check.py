#!/usr/bin/env python
"""Orbital-sharded evaluation with the fused peer-memory gather (PeerGather)
under torchrun: every rank evaluates all positions on its spline slice and
stores it straight into rank 0's [P][S][N] buffer; rank 0 then checks the
result bitwise against a full-N evaluation and, when every rank has its own
GPU, against the NCCL all-gather baseline (gather_orbital_blocks), timing both.

    torchrun --nproc-per-node K --master-addr 127.0.0.1 scripts/peer_gather_check.py \\
        [--grid 24] [--splines 200] [--positions 3000] [--kind vgh] [--dtype f32]

Ranks may share one GPU (the check then runs over gloo; kernels never wait on
each other, they only write disjoint lanes of rank 0's buffer).
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import torch.distributed as dist

    from paper_1611_02665_b200 import DeviceTable, evaluate
    from paper_1611_02665_b200.grid import unit_cell_grid
    from paper_1611_02665_b200.multi import OrbitalPartition, PeerGather, gather_orbital_blocks

    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=24)
    ap.add_argument("--splines", type=int, default=200)
    ap.add_argument("--positions", type=int, default=3000)
    ap.add_argument("--kind", default="vgh")
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--kpower", action="store_true", help="evaluate on the opt-in k-power table form")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    ngpu = torch.cuda.device_count()
    own_gpu = ngpu >= world
    dev = torch.device("cuda", local if own_gpu else 0)
    torch.cuda.set_device(dev)
    backend = "nccl" if own_gpu else "gloo"
    if world > 1:
        dist.init_process_group(backend, device_id=dev if backend == "nccl" else None)

    grid = unit_cell_grid(args.grid)
    q = 4 if args.dtype == "f32" else 2
    part = OrbitalPartition.make(args.splines, world, quantum=max(q, 16))
    if args.dtype == "f32":
        full = DeviceTable.random(grid, args.splines, seed=7, device=dev)
    else:
        full = DeviceTable.normal_f64(grid, args.splines, seed=7, device=dev)
    lo, hi = part.local(rank)
    mine = full.slice_orbitals(lo, hi)
    if args.kpower:
        full.with_kpower()
        mine.with_kpower()
    rng = np.random.default_rng(11)
    pos = torch.from_numpy(rng.random((args.positions, 3)) * 2.0 - 0.5).to(dev)

    form = "kpower" if args.kpower else "auto"
    pg = PeerGather(part, args.kind, args.positions, full.dtype, root=0, device=dev)
    res = {"world": world, "backend": backend, "ranks_share_gpu": not own_gpu, "bounds": part.bounds}
    from paper_1611_02665_b200.kernels import eval_form

    res["form"] = eval_form(mine, args.kind, args.positions, form=form)
    # two different position sets through the same gather buffer: the second
    # call must wait for the root to finish with the first call's view
    pos2 = torch.from_numpy(rng.random((args.positions, 3)) * 3.0 - 1.0).to(dev)
    bitwise = True
    for p in (pos2, pos):
        got = pg.evaluate(mine, p, form=form)
        if rank == 0:
            want = evaluate(full, args.kind, p, form=form)[:, :, : args.splines]
            bitwise &= bool(torch.equal(got, want))
    if rank == 0:
        res["peer_bitwise"] = bitwise

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            fn()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / args.reps

    res["peer_ms"] = timed(lambda: pg.evaluate(mine, pos, form=form))
    if own_gpu:
        def nccl_path():
            block = evaluate(mine, args.kind, pos, form=form)[:, :, : hi - lo]
            return gather_orbital_blocks(block, part, root=0) if world > 1 else block
        out = nccl_path()
        if rank == 0:
            res["nccl_bitwise"] = bool(torch.equal(out, want))
        res["nccl_ms"] = timed(nccl_path)
    if world > 1:
        dist.barrier()
    if rank == 0:
        print(json.dumps(res), flush=True)
        ok = res["peer_bitwise"] and res.get("nccl_bitwise", True)
    else:
        ok = True
    if world > 1:
        dist.destroy_process_group()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())

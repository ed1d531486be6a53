"""Multi-GPU partitioning: one process per GPU over torch.distributed.

Two modes, both without a collective on the evaluation path:

* walker-sharded -- the reference's walker-level parallelism (driver.py:298-346)
  across GPUs: every rank holds the full table and evaluates a contiguous,
  walker-aligned share of the positions.  Outputs stay on their rank.
* orbital-sharded -- the reference's nested tile parallelism (driver.py:349-434,
  tile_table coeffs.py:197-210) across GPUs: rank r holds splines
  [lo_r, hi_r) and evaluates every position for that slice.  Only when the
  caller needs full-N outputs on one device are the slices gathered along N
  with NCCL (all-gather into [world][P][S][n_max] + a local permute), which is
  the one exchange step of the path.

The partition/gather helpers take plain tensors so they also run on CPU with
the gloo backend (tests/test_multi_gloo.py); the evaluation itself is the
CUDA path (kernels.evaluate).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def balanced_bounds(n: int, parts: int, quantum: int = 1):
    """Split range(n) into `parts` contiguous [lo, hi) pieces whose sizes are
    multiples of `quantum` (except possibly the last) and differ by at most
    one quantum."""
    if parts < 1:
        raise ValueError("parts must be >= 1")
    units = -(-n // quantum)
    base, extra = divmod(units, parts)
    out, lo = [], 0
    for r in range(parts):
        size = (base + (1 if r < extra else 0)) * quantum
        hi = min(n, lo + size)
        out.append((lo, hi))
        lo = hi
    return out


def walker_shard(n_walkers: int, world: int, rank: int) -> range:
    """Walkers owned by `rank` (contiguous, balanced)."""
    lo, hi = balanced_bounds(n_walkers, world)[rank]
    return range(lo, hi)


def position_shard(n_positions: int, moves_per_walker: int, world: int, rank: int) -> slice:
    """Walker-aligned slice of a [walkers * moves] position array."""
    w = walker_shard(n_positions // moves_per_walker, world, rank)
    return slice(w.start * moves_per_walker, w.stop * moves_per_walker)


@dataclass(frozen=True)
class OrbitalPartition:
    """Spline ranges per rank for the orbital-sharded mode."""

    n_splines: int
    bounds: tuple  # ((lo, hi), ...) per rank

    @classmethod
    def make(cls, n_splines: int, world: int, quantum: int = 16):
        return cls(n_splines, tuple(balanced_bounds(n_splines, world, quantum)))

    @property
    def world(self) -> int:
        return len(self.bounds)

    @property
    def n_max(self) -> int:
        return max(hi - lo for lo, hi in self.bounds)

    def local(self, rank: int):
        return self.bounds[rank]


def gather_orbital_blocks(local, part: OrbitalPartition, group=None, root=None):
    """Gather per-rank orbital blocks [P][S][n_r] into [P][S][N].

    NCCL all-gather of equal-size padded blocks [P][S][n_max] into
    [world][P][S][n_max], then a local permute onto the spline axis.  With
    `root` set only that rank materialises the result (others return None);
    with root=None every rank gets it.
    """
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    if world != part.world:
        raise ValueError(f"partition has {part.world} ranks, group has {world}")
    P, S, n_local = local.shape
    lo, hi = part.local(rank)
    if n_local != hi - lo:
        raise ValueError(f"rank {rank} block has {n_local} splines, partition says {hi - lo}")
    nmax = part.n_max
    send = local if n_local == nmax else torch.nn.functional.pad(local, (0, nmax - n_local))
    send = send.contiguous()
    buf = torch.empty((world * P, S, nmax), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(buf, send, group=group)
    buf = buf.view(world, P, S, nmax)
    if root is not None and rank != root:
        return None
    out = torch.empty((P, S, part.n_splines), dtype=local.dtype, device=local.device)
    for r, (a, b) in enumerate(part.bounds):
        out[:, :, a:b] = buf[r, :, :, : b - a]
    return out


def evaluate_walker_sharded(table, kind, positions, moves_per_walker: int, group=None, **kw):
    """Evaluate this rank's walker share of `positions` (table replicated).
    Returns (slice of positions, outputs [P_local][S][lanes])."""
    import torch.distributed as dist

    from .kernels import evaluate

    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    sl = position_shard(len(positions), moves_per_walker, world, rank)
    return sl, evaluate(table, kind, positions[sl], **kw)


def evaluate_orbital_sharded(local_table, kind, positions, part: OrbitalPartition, group=None,
                             root=None, **kw):
    """Every rank evaluates all positions on its spline slice; the slices
    are then gathered along N (gather_orbital_blocks).  `local_table` is the
    rank's DeviceTable holding splines part.local(rank).  Returns the full
    [P][S][N] outputs (on `root`, or everywhere with root=None) and the local
    evaluation result."""
    from .kernels import evaluate

    local = evaluate(local_table, kind, positions, **kw)
    if local_table.tiled:
        block = local.index_select(2, local_table.lane_index())
    else:
        block = local[:, :, : local_table.n_splines]
    full = gather_orbital_blocks(block, part, group=group, root=root)
    return full, local


def shard_table_for_rank(full_table, part: OrbitalPartition, rank: int, tile_size=None):
    """The rank's DeviceTable slice of a full DeviceTable (single-node helper)."""
    lo, hi = part.local(rank)
    return full_table.slice_orbitals(lo, hi, tile_size=tile_size)


def split_array(a: np.ndarray, bounds):
    return [a[..., lo:hi] for lo, hi in bounds]

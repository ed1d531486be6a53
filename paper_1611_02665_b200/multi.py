"""Multi-GPU partitioning: one process per GPU over torch.distributed.

Two modes, both without a collective on the evaluation path:

* walker-sharded -- the reference's walker-level parallelism (driver.py:298-346)
  across GPUs: every rank holds the full table and evaluates a contiguous,
  walker-aligned share of the positions.  Outputs stay on their rank.
* orbital-sharded -- the reference's nested tile parallelism (driver.py:349-434,
  tile_table coeffs.py:197-210) across GPUs: rank r holds splines
  [lo_r, hi_r) and evaluates every position for that slice.  Only when the
  caller needs full-N outputs on one device are the slices gathered along N,
  the one exchange step of the path: fused into the kernel's own output
  stores over peer memory (PeerGather, spo_eval_lanes), or with NCCL
  (gather_orbital_blocks: all-gather into [world][P][S][n_max] + a local
  permute) as the baseline.

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


def sum_ratio_partials(partial, group=None, root=None):
    """The exchange step of the sharded consumer: every rank holds the [P][S]
    fp64 partial contraction over its own spline slice; their sum over the
    ranks is the full contraction.  An all-reduce (root=None: the result on
    every rank, in place) or a reduce onto `root` (other ranks return None).
    P * S * 8 bytes per rank, against P * S * N * sizeof(T) for gathering the
    streams themselves (config 5: 1.7 MB against 132.5 GB per step)."""
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return partial
    if root is None:
        dist.all_reduce(partial, op=dist.ReduceOp.SUM, group=group)
        return partial
    dist.reduce(partial, dst=root, op=dist.ReduceOp.SUM, group=group)
    return partial if dist.get_rank(group) == root else None


def evaluate_ratios_orbital_sharded(local_table, kind, positions, coef_local, group=None, root=None, **kw):
    """Orbital-sharded fused consumer (the scalable alternative to gathering
    the full [P][S][N] outputs onto one GPU): every rank
    contracts every position's streams over its own spline slice with its slice
    of the coefficient rows (kernels.evaluate_ratios: the outputs are never
    written), then the (P, S) fp64 partials are summed over the ranks.
    coef_local: (P, n_local) -- columns part.local(rank) of the full (P, N)
    coefficients.  The slice tables need 512-byte rows (tiled, as
    slice_orbitals' default tile_size="auto" makes them), the ratio kernel's
    own contract.  Returns the (P, S) float64 ratios (on `root`, or everywhere
    with root=None)."""
    from .kernels import evaluate_ratios

    partial = evaluate_ratios(local_table, kind, positions, coef_local, **kw)
    return sum_ratio_partials(partial, group=group, root=root)


def _lane_quantum(dtype) -> int:
    """Output lanes per 16-byte store (fp32: 4, fp64: 2)."""
    return 16 // np.dtype(dtype).itemsize


def check_peer_partition(part: OrbitalPartition, dtype) -> None:
    """Every rank's first spline must start a 16-byte lane vector of the
    root's rows, so its stores stay aligned and never touch a neighbour's
    lanes (the last lane vector of a slice is stored lane by lane)."""
    q = _lane_quantum(dtype)
    for r, (lo, _hi) in enumerate(part.bounds):
        if lo % q:
            raise ValueError(f"rank {r} starts at spline {lo}, not a multiple of {q}: "
                             f"use OrbitalPartition.make(..., quantum={q}) or a multiple")


class PeerGather:
    """Fused evaluate + gather along N over peer memory (orbital-sharded mode,
    SURVEY.md 8(e)).

    The root allocates the full [capacity][S][Npad] output once and shares it
    with every rank of `group` as a CUDA IPC handle (torch's CUDA tensor
    reduction, sent with broadcast_object_list).  evaluate() then runs each
    rank's kernel on its own GPU with spo_eval_lanes: the rank's spline slice
    [lo, hi) is stored straight into the root's buffer at lane offset lo, so
    the transfer rides on the kernel's own output stores over NVLink, overlapped
    with the math tile by tile -- no gather buffer, no all-gather of padded
    blocks, no permute (compare gather_orbital_blocks, the NCCL baseline).
    Completion: every rank synchronises its stream, then a group barrier;
    after it the root's view holds all N splines.  Kernels never wait on each
    other.
    """

    def __init__(self, part: OrbitalPartition, kind, capacity: int, dtype, group=None, root: int = 0,
                 device=None):
        import torch
        import torch.distributed as dist

        from .kernels import as_kind

        self.part, self.kind, self.group, self.root = part, as_kind(kind), group, root
        self.dtype = np.dtype(dtype)
        self.capacity = int(capacity)
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        if world != part.world:
            raise ValueError(f"partition has {part.world} ranks, group has {world}")
        check_peer_partition(part, self.dtype)
        q = _lane_quantum(self.dtype)
        self.npad = -(-part.n_splines // q) * q
        S = self.kind.output_streams_soa
        tdt = torch.float64 if self.dtype == np.float64 else torch.float32
        device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        handle = [None]
        if self.rank == root:
            self.buf = torch.empty((self.capacity, S, self.npad), dtype=tdt, device=device)
            if world > 1:
                from torch.multiprocessing.reductions import reduce_tensor

                handle = [reduce_tensor(self.buf)]
        if world > 1:
            dist.broadcast_object_list(handle, src=root, group=group)
            if self.rank != root:
                fn, args = handle[0]
                self.buf = fn(*args)  # IPC mapping of the root's buffer in this process

    def evaluate(self, local_table, positions, **kw):
        """Evaluate this rank's spline slice at every position into the root's
        buffer.  Returns the root's [P][S][N] view on the root, None elsewhere.
        The view is valid until the next evaluate() call on this gather (the
        next call waits for the root's stream, then overwrites it)."""
        import torch
        import torch.distributed as dist

        from .device import as_device_table
        from .errors import ContractError
        from .kernels import _positions_tensor, evaluate

        dt = as_device_table(local_table)
        lo, hi = self.part.local(self.rank)
        if dt.n_splines != hi - lo:
            raise ContractError(f"rank {self.rank} table has {dt.n_splines} splines, partition says {hi - lo}")
        if np.dtype(dt.dtype) != self.dtype:
            raise ContractError("table dtype differs from the gather buffer's")
        if not dt.lanes_are_splines:
            raise ContractError("spo_eval_lanes needs lanes == spline indices (untiled, or tiles "
                                "without padding lanes)")
        pos = _positions_tensor(positions, dt.device)
        P = pos.shape[0]
        if P > self.capacity:
            raise ContractError(f"{P} positions exceed the gather buffer's capacity {self.capacity}")
        multi_rank = dist.is_initialized() and dist.get_world_size(self.group) > 1
        if multi_rank:
            # Reuse contract: the view returned by the previous call stays valid
            # until the next call.  The root drains its stream (any work it
            # queued on that view) and every rank waits for it here, so no
            # rank's stores can overwrite a buffer the root is still reading.
            if self.rank == self.root:
                torch.cuda.current_stream(dt.device).synchronize()
            dist.barrier(group=self.group)
        if hi > lo:
            evaluate(dt, self.kind, pos, self.buf[:P, :, lo:], lane_limit=hi - lo, **kw)
        if multi_rank:
            torch.cuda.current_stream(dt.device).synchronize()
            dist.barrier(group=self.group)
        return self.buf[:P, :, : self.part.n_splines] if self.rank == self.root else None


def shard_table_for_rank(full_table, part: OrbitalPartition, rank: int, tile_size=None):
    """The rank's DeviceTable slice of a full DeviceTable (single-node helper)."""
    lo, hi = part.local(rank)
    return full_table.slice_orbitals(lo, hi, tile_size=tile_size)


def split_array(a: np.ndarray, bounds):
    return [a[..., lo:hi] for lo, hi in bounds]

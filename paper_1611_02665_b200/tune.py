"""Device-side AoSoA tile-size autotuner.

Mirrors the reference's tuner (metrics.py:241-314): scan tile sizes doubling
up to N, score each by median throughput (orbital-evals/s) over `repeats`
timed repetitions, return the argmax with ties broken toward the larger tile.
Differences, all B200-driven: candidates start at 32 lanes (the 128-byte row
quantum) instead of 16; timing is CUDA events around batched launches on the
device table instead of a single-threaded host loop; the probe batch is a
walker-position stream of `n_positions` (default 65,536) so that the tile
slice, not launch latency, decides.
"""
from __future__ import annotations

import statistics
from dataclasses import dataclass

import numpy as np

from .device import DeviceTable
from .errors import ConfigError
from .kernels import as_kind, evaluate
from .workloads import walker_positions


@dataclass(frozen=True)
class TuneResult:
    scanned: tuple
    throughputs: tuple
    best_tile: int
    best_throughput: float


def tile_candidates(n_splines: int, quantum: int = 32) -> list:
    """quantum, 2*quantum, ... doubling while below N, then N (untiled)."""
    if n_splines < quantum:
        raise ConfigError(f"n_splines={n_splines} < {quantum}: tuning does not apply, run untiled")
    sizes, nb = [], quantum
    while nb < n_splines:
        sizes.append(nb)
        nb *= 2
    sizes.append(n_splines)
    return sizes


def retile(table: DeviceTable, tile_size) -> DeviceTable:
    """The same coefficients in another AoSoA tiling (device-side repack)."""
    return table.slice_orbitals(0, table.n_splines, tile_size=tile_size)


def tune_tile_size(table: DeviceTable, kind, n_positions: int = 1 << 16, repeats: int = 3,
                   seed: int = 1, candidates=None, kpower=False) -> TuneResult:
    """Scan tilings of `table` for `kind`; returns the argmax (ties -> larger tile).
    kpower: time every candidate on the opt-in k-power table form
    (form="kpower") instead of the default B-spline form."""
    import torch

    kind = as_kind(kind)
    cands = list(candidates) if candidates is not None else tile_candidates(table.n_splines)
    moves = 256
    walkers = max(1, -(-n_positions // moves))
    pos_np = walker_positions(seed, range(walkers), 0, kind.value, moves, table.grid)[:n_positions]
    pos = torch.from_numpy(np.ascontiguousarray(pos_np)).to(table.device)
    scores = []
    best_tile, best = 0, float("-inf")
    stream = torch.cuda.current_stream(table.device)
    for nb in cands:
        t = retile(table, None if nb >= table.n_splines else nb)
        if kpower:
            t.with_kpower()
        out = torch.empty((pos.shape[0], kind.output_streams_soa, t.lanes), dtype=t.data.dtype,
                          device=t.device)
        form = "kpower" if kpower else "bspline"
        evaluate(t, kind, pos, out, check=False, form=form)  # warm-up
        reps = []
        for _ in range(repeats):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            evaluate(t, kind, pos, out, check=False, form=form)
            e1.record(stream)
            e1.synchronize()
            reps.append(pos.shape[0] * table.n_splines / (e0.elapsed_time(e1) * 1e-3))
        score = statistics.median(reps)
        scores.append(score)
        if score >= best:  # ascending scan: >= prefers the larger tile
            best_tile, best = nb, score
        del t, out
    return TuneResult(tuple(cands), tuple(scores), best_tile, best)

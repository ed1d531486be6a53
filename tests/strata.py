"""Stratified oracle samples for the full-size parity tests (SURVEY.md 4.3-3,
VERDICT r1 "Next round" 2).

A sample of a launch's positions that contains
* one position from every 4x4x4-cell block of the grid that holds any
  (64^3: 4096 blocks, 48^3: 1728),
* the first and last position of line-kernel runs -- the kernel sorts a
  launch's positions by (spatial block, j0, k0, i0) and hands them out in
  runs of 64 (csrc/spo_eval_line.cu line_keys_kernel, BPL); the order is
  restated here with a stable sort, as cub's radix sort is stable,
* random positions up to `n_min`.
"""
import numpy as np

import oracle

BPL = 64  # positions per line-kernel run (SPO_LINE_BPL)


def cells(pos, grid):
    """(i0, j0, k0) int64 arrays of the reference mapping (grid.py:109-121)."""
    out = []
    for a, (cnt, d) in enumerate(zip(grid.counts, grid.spacings)):
        i, _ = oracle.map_axis(pos[:, a], 1.0 / d, cnt)
        out.append(np.asarray(i, dtype=np.int64))
    return out


def line_order(pos, grid, nbk=(4, 4, 4)):
    """The line kernel's sorted order of one launch's positions."""
    i0, j0, k0 = cells(pos, grid)
    n = grid.counts
    b = ((i0 * nbk[0] // n[0]) * nbk[1] + j0 * nbk[1] // n[1]) * nbk[2] + k0 * nbk[2] // n[2]
    key = (b << 24) | (j0 << 16) | (k0 << 8) | i0
    return np.argsort(key, kind="stable")


def stratified_sample(pos, grid, n_min=2048, seed=0, runs=192, launch=None):
    """Sorted unique indices into `pos`.  `launch`: positions per launch (the
    run boundaries are computed per launch chunk); None = one launch."""
    rng = np.random.default_rng(seed)
    P = pos.shape[0]
    i0, j0, k0 = cells(pos, grid)
    block = ((i0 // 4) * ((grid.ny + 3) // 4) + j0 // 4) * ((grid.nz + 3) // 4) + k0 // 4
    perm = rng.permutation(P)
    _, first = np.unique(block[perm], return_index=True)
    pick = [perm[first]]
    launch = launch or P
    for lo in range(0, P, launch):
        hi = min(P, lo + launch)
        order = line_order(pos[lo:hi], grid) + lo
        n_runs = -(-(hi - lo) // BPL)
        chosen = np.unique(np.concatenate([[0, n_runs - 1], rng.choice(n_runs, min(runs, n_runs), replace=False)]))
        starts = chosen * BPL
        ends = np.minimum(starts + BPL, hi - lo) - 1
        pick += [order[starts], order[ends]]
    sel = np.unique(np.concatenate(pick))
    if sel.size < n_min:
        rest = np.setdiff1d(np.arange(P), sel)
        sel = np.union1d(sel, rng.choice(rest, min(rest.size, n_min - sel.size), replace=False))
    return sel

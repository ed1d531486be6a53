"""The line/window prologue's plane sequence (csrc/spo_eval_line.cu,
line_runs_kernel): the sequential rule of round 1 and the warp-scan form the
kernel now runs (segmented max of i0+3, prefix sum of appended-plane counts)
restated in numpy and checked against each other on random sorted runs.  The
GPU kernels themselves are checked bitwise against the per-position kernel
(tests/test_gpu_line.py, test_gpu_stress.py); this pins the algorithm."""
import numpy as np
import pytest


def serial(cells, win):
    """cells: (n, 3) int (i0, j0, k0), i0 < 0 = non-finite.  -> (s, planes)."""
    cj = ck = last = -1
    planes, s_out = [], []
    for i0, j0, k0 in cells:
        s = 0
        if i0 >= 0:
            wj, wk = win * (j0 // win), win * (k0 // win)
            same = wj == cj and wk == ck
            if same and i0 <= last:
                s = len(planes) - 1 - (last - i0)
                lo = last + 1
            else:
                s = len(planes)
                lo = i0
            planes += [(t, wj, wk) for t in range(lo, i0 + 4)]
            if not same or i0 + 3 > last:
                last = i0 + 3
            cj, ck = wj, wk
        s_out.append(s)
    return s_out, planes


def scanned(cells, win):
    """The kernel's formulation (finite positions first, as the sort leaves them)."""
    n = len(cells)
    ok = cells[:, 0] >= 0
    assert not (~ok[:-1] & ok[1:]).any(), "non-finite positions must form a suffix"
    i0 = cells[:, 0]
    wj, wk = win * (cells[:, 1] // win), win * (cells[:, 2] // win)
    same = np.zeros(n, bool)
    same[1:] = ok[1:] & (wj[1:] == wj[:-1]) & (wk[1:] == wk[:-1])
    v = i0 + 3
    run = np.empty(n, np.int64)  # segmented inclusive max (a new line starts a segment)
    for q in range(n):
        run[q] = v[q] if (q == 0 or not same[q]) else max(run[q - 1], v[q])
    lastp = np.concatenate([[-1], run[:-1]])
    share = same & (i0 <= lastp)
    lo = np.where(share, lastp + 1, i0)
    cnt = np.where(~ok, 0, np.where(share, np.maximum(0, i0 + 3 - lastp), 4))
    nxt = np.concatenate([[0], np.cumsum(cnt)[:-1]])
    s = np.where(~ok, 0, np.where(share, nxt - 1 - (lastp - i0), nxt))
    planes = [(int(lo[q] + t), int(wj[q]), int(wk[q])) for q in range(n) for t in range(cnt[q])]
    return [int(x) for x in s], planes


@pytest.mark.parametrize("win", [1, 2, 3])
@pytest.mark.parametrize("density", [0.1, 1.0, 8.0])
def test_scan_form_equals_sequential_rule(win, density):
    rng = np.random.default_rng(int(density * 10) + win)
    n_grid = 16
    for trial in range(40):
        P = 64
        span = max(1, int(P / density))
        cells = rng.integers(0, n_grid, (P, 3))
        cells[:, 1] = rng.integers(0, max(1, min(n_grid, span // n_grid + 1)), P)
        # the sort order of the kernel's keys: (window/line, i0); invalid last
        key = (win * (cells[:, 1] // win)) * 1000 + (win * (cells[:, 2] // win))
        order = np.lexsort((cells[:, 0], key))
        cells = cells[order]
        n_bad = int(rng.integers(0, 3)) if trial % 4 == 0 else 0
        if n_bad:
            cells[-n_bad:, 0] = -1
        assert scanned(cells, win) == serial(cells, win)


def groups_serial(cells, vgroup):
    """Cell-aligned V groups, the rule: a group starts at every new cell (a
    non-finite position is a cell of its own) and after every vgroup positions
    of a cell.  -> the start position of each group."""
    starts, prev, in_cell = [], None, 0
    for q, (i0, j0, k0) in enumerate(cells):
        cell = (int(i0), int(j0), int(k0))
        if q == 0 or i0 < 0 or cell != prev:
            in_cell = 0
        if in_cell % vgroup == 0:
            starts.append(q)
        in_cell += 1
        prev = cell
    return starts


def groups_scanned(cells, vgroup):
    """line_runs_kernel's form: two positions per lane; new-cell flags, the
    start of a position's cell by an inclusive max scan over the lanes, the
    group number by a prefix sum of the group-start flags."""
    nb = len(cells)
    lanes = 32
    pad = np.full((2 * lanes, 3), -7)
    pad[:nb] = cells
    ok = np.zeros(2 * lanes, bool)
    ok[:nb] = cells[:, 0] >= 0
    a, b = pad[0::2], pad[1::2]  # the lane's two positions
    prev_b = np.roll(b, 1, axis=0)
    nc0 = (np.arange(lanes) == 0) | ~ok[0::2] | (a != prev_b).any(axis=1)
    nc1 = ~ok[1::2] | (b != a).any(axis=1)
    cs = np.where(nc1, 2 * np.arange(lanes) + 1, np.where(nc0, 2 * np.arange(lanes), -1))
    d = 1
    while d < lanes:  # the shuffle scan, step by step
        o = np.concatenate([np.full(d, -1), cs[:-d]])
        cs = np.where(np.arange(lanes) >= d, np.maximum(cs, o), cs)
        d <<= 1
    csb = np.concatenate([[-1], cs[:-1]])
    st0 = np.where(nc0, 2 * np.arange(lanes), csb)
    st1 = np.where(nc1, 2 * np.arange(lanes) + 1, st0)
    q0, q1 = 2 * np.arange(lanes), 2 * np.arange(lanes) + 1
    gf0 = (q0 < nb) & ((q0 - st0) % vgroup == 0)
    gf1 = (q1 < nb) & ((q1 - st1) % vgroup == 0)
    gi = np.cumsum(gf0.astype(int) + gf1.astype(int))
    g1 = gi - 1
    g0 = g1 - gf1.astype(int)
    gs = np.full(2 * lanes, 0xFF)
    gs[g0[gf0]] = q0[gf0]
    gs[g1[gf1]] = q1[gf1]
    return [int(x) for x in gs if x != 0xFF]


@pytest.mark.parametrize("vgroup", [2, 3, 4, 5])
@pytest.mark.parametrize("density", [1.0, 4.0, 16.0])
def test_cell_aligned_group_starts(vgroup, density):
    """The V launch's cell-aligned groups (SPO_VCELL): the warp-scan form equals
    the sequential rule on full and ragged runs, with non-finite positions."""
    rng = np.random.default_rng(vgroup * 100 + int(density))
    for trial in range(60):
        nb = 64 if trial % 3 else int(rng.integers(1, 65))
        n_cells = max(1, int(nb / density))
        ids = np.sort(rng.integers(0, n_cells, nb))
        cells = np.stack([ids % 7, (ids // 7) % 5, ids // 35], axis=1)
        cells = cells[np.lexsort((cells[:, 0], cells[:, 2], cells[:, 1]))]
        n_bad = int(rng.integers(1, 4)) if trial % 5 == 0 else 0
        if n_bad:
            cells[-min(n_bad, nb):, 0] = -1
        got = groups_scanned(cells, vgroup)
        assert got == groups_serial(cells, vgroup)
        sizes = np.diff(got + [nb])
        assert sizes.min() >= 1 and sizes.max() <= vgroup

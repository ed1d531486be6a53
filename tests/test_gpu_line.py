"""The line-window kernel (spo_eval_line.cu: stencil planes shared along grid
lines) is bitwise identical to the per-position TMA kernel and the generic
kernel on every input class: kinds, fp32/fp64, tiled/untiled tables, ragged
runs, duplicate cells, a single line, non-finite positions, out_index,
lane_limit, and grids too large for its sort key (fallback) -- and so is its
window variant for sparse batches.  SPO_LINE=1/2/0 forces the line kernel,
the window variant or the per-position kernel (read on every call)."""
import numpy as np
import pytest

import oracle
from paper_1611_02665_b200 import DeviceTable, DomainError, KernelKind, evaluate, streams
from paper_1611_02665_b200.grid import GridSpec, unit_cell_grid

pytestmark = pytest.mark.gpu


def _both(monkeypatch, dt, kind, pos, **kw):
    """(line, per-position) outputs; the window variant must equal both."""
    monkeypatch.setenv("SPO_LINE", "1")
    a = evaluate(dt, kind, pos, pipeline=True, **kw).clone()
    monkeypatch.setenv("SPO_LINE", "2")
    w = evaluate(dt, kind, pos, pipeline=True, **kw).clone()
    monkeypatch.setenv("SPO_LINE", "0")
    b = evaluate(dt, kind, pos, pipeline=True, **kw)
    monkeypatch.delenv("SPO_LINE")
    assert _eq(w, b), "window variant differs from the per-position kernel"
    return a, b


def _eq(a, b):
    import torch

    return bool(torch.equal(a.nan_to_num(123.0), b.nan_to_num(123.0)))


@pytest.mark.parametrize("kind", ["v", "vgl", "vgh"])
@pytest.mark.parametrize("tile", ["auto", None])
def test_line_bitwise_fp32(monkeypatch, kind, tile):
    dt = DeviceTable.random(unit_cell_grid(20), 512, seed=5, tile_size=tile)
    pos = np.random.default_rng(2).random((30000 + 17, 3)) * 3.0 - 1.0  # ragged last run, wrapped inputs
    a, b = _both(monkeypatch, dt, kind, pos)
    assert _eq(a, b)


@pytest.mark.parametrize("kind", ["v", "vgh"])
def test_line_bitwise_fp64(monkeypatch, kind):
    dt = DeviceTable.normal_f64(unit_cell_grid(16), 128, seed=5)
    pos = np.random.default_rng(3).random((20000, 3))
    a, b = _both(monkeypatch, dt, kind, pos)
    assert _eq(a, b)


def test_line_matches_oracle(monkeypatch):
    """Anchor: the line path against the fp64 oracle at 1e-5 * sum|w*c|."""
    grid = unit_cell_grid(12)
    dt = DeviceTable.random(grid, 256, seed=9)
    pos = np.random.default_rng(4).random((4000, 3))
    monkeypatch.setenv("SPO_LINE", "1")
    got = streams(evaluate(dt, "vgh", pos, pipeline=True), dt, "vgh")
    names = KernelKind("vgh").stream_names
    sample = np.arange(0, 4000, 37)
    ref, scale = oracle.eval_f64("vgh", dt.reference_soa(), 256, grid.spacings, pos[sample])
    g = np.stack([got[n].cpu().numpy()[sample] for n in names], axis=1)
    ok, worst = oracle.tolerance_check(g, ref, scale, 1e-5)
    assert ok, worst


def test_line_duplicate_cells_and_single_line(monkeypatch):
    rng = np.random.default_rng(5)
    dt = DeviceTable.random(unit_cell_grid(24), 256, seed=1)
    # 40 cells, ~250 positions each: runs made of repeated cells
    centers = rng.integers(0, 24, size=(40, 3)) / 24.0
    dup = centers[rng.integers(0, 40, size=10000)] + rng.random((10000, 3)) * (0.9 / 24)
    a, b = _both(monkeypatch, dt, "vgh", dup)
    assert _eq(a, b)
    # every position on one grid line (fixed y, z): maximal plane sharing
    line = np.stack([rng.random(8000) * 2 - 0.5, np.full(8000, 0.31), np.full(8000, 0.77)], axis=1)
    a, b = _both(monkeypatch, dt, "vgl", line)
    assert _eq(a, b)


def test_line_nonfinite_positions(monkeypatch):
    import torch

    dt = DeviceTable.random(unit_cell_grid(16), 128, seed=2)
    pos = np.random.default_rng(6).random((5000, 3))
    pos[[3, 777, 4999], [0, 1, 2]] = [np.nan, np.inf, -np.inf]
    pos = torch.from_numpy(pos).cuda()  # device input: checked by the kernels' status flag
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    a, b = _both(monkeypatch, dt, "vgh", pos, status=st, check=False)
    assert _eq(a, b) and int(st.item()) == 1
    assert bool(torch.isnan(a[777]).all()) and not bool(torch.isnan(a[778]).any())
    monkeypatch.setenv("SPO_LINE", "1")
    with pytest.raises(DomainError):
        evaluate(dt, "vgh", pos, pipeline=True)


def test_line_out_index_and_lane_limit(monkeypatch):
    import torch

    dt = DeviceTable.random(unit_cell_grid(16), 256, seed=3)
    P = 6000
    pos = np.random.default_rng(7).random((P, 3))
    perm = torch.from_numpy(np.random.default_rng(8).permutation(P)).cuda()
    outs = []
    for v in ("1", "0"):
        monkeypatch.setenv("SPO_LINE", v)
        o = torch.full((P, 10, dt.lanes), 5.0, device="cuda")
        evaluate(dt, "vgh", pos, o, out_index=perm, pipeline=True)
        buf = torch.full((P, 10, 300), 5.0, device="cuda")
        evaluate(dt, "vgh", pos, buf[:, :, 4:], pipeline=True, lane_limit=201)
        outs.append((o, buf))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    assert bool((outs[0][1][:, :, 205:] == 5.0).all())


def test_line_wide_and_ragged_tiles(monkeypatch):
    dt = DeviceTable.random(unit_cell_grid(12), 1000, seed=4)  # last tile partially filled
    pos = np.random.default_rng(9).random((7000, 3))
    a, b = _both(monkeypatch, dt, "vgh", pos)
    assert _eq(a, b)


def test_line_large_grid_falls_back(monkeypatch):
    """Axes above 256 cells do not fit the sort key: the TMA kernel runs."""
    grid = GridSpec(300, 4, 4, 1 / 300, 0.25, 0.25)
    dt = DeviceTable.random(grid, 32, seed=1)
    pos = np.random.default_rng(1).random((9000, 3))
    a, b = _both(monkeypatch, dt, "v", pos)
    assert _eq(a, b)


def test_line_large_batch(monkeypatch):
    """2.1M positions (64 per cell, many full runs of one cell): the radix
    sort's double buffers and the exact workspace query at scale."""
    import torch

    from paper_1611_02665_b200.kernels import eval_path

    dt = DeviceTable.random(unit_cell_grid(32), 128, seed=6)
    P = 2_100_000
    assert eval_path(dt, "vgl", P) == "line"
    pos = torch.from_numpy(np.random.default_rng(10).random((P, 3))).cuda()
    a, b = _both(monkeypatch, dt, "vgl", pos)
    assert _eq(a, b)


@pytest.mark.parametrize("dtype,tile", [("f32", 256), ("f64", None)])
def test_line_noncubic_grid_and_tilings(monkeypatch, dtype, tile):
    """Non-cubic grid with non-unit spacings; fp32 tiles of 256 lanes (two
    units per tile row) and an untiled fp64 table."""
    grid = GridSpec(12, 20, 7, 0.5, 0.25, 1.0 / 7)
    dt = (DeviceTable.random(grid, 512, seed=2, tile_size=tile) if dtype == "f32"
          else DeviceTable.normal_f64(grid, 128, seed=2, tile_size=tile))
    pos = np.random.default_rng(12).random((9000, 3)) * np.array([6.0, 5.0, 1.0]) * 1.5 - 1.0
    a, b = _both(monkeypatch, dt, "vgh", pos)
    assert _eq(a, b)


def test_line_edge_coordinates(monkeypatch):
    """The reference's awkward coordinates (golden mapping set: +-0, denormals,
    +-1e308, +-1e15, cell boundaries, negatives) through the line kernel."""
    import os

    xs = np.load(os.path.join(os.path.dirname(__file__), "golden", "mapping.npz"))["xs"]
    grid = GridSpec(20, 24, 28, 0.05, 1 / 24, 1 / 28)
    dt = DeviceTable.random(grid, 128, seed=4)
    rng = np.random.default_rng(13)
    pos = np.stack([rng.choice(xs, 20000), rng.choice(xs, 20000), rng.random(20000)], axis=1)
    a, b = _both(monkeypatch, dt, "vgh", pos)
    assert _eq(a, b)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_v_group_sizes_and_assignment(monkeypatch, dtype):
    """Every V group size the launcher accepts (SPO_VGROUP, including the ones
    the ring cannot hold, which fall back), on the line kernel and the 2 x 1
    window, with the groups handed out dynamically (default) and statically
    (SPO_VDYN=0), the same-cell path on and off, the groups fixed or aligned to
    cells by the prologue (SPO_VCELL): bitwise equal to the per-position kernel.  The timeout is the deadlock check (a ring smaller
    than 4 VGROUP + PBATCH - 1 planes would hang; ring_min in the kernel)."""
    grid = unit_cell_grid(12)
    dt = DeviceTable.random(grid, 256, seed=3) if dtype == "f32" else DeviceTable.normal_f64(grid, 128, seed=3)
    rng = np.random.default_rng(8)
    dense = rng.random((12 ** 3 * 9 + 5, 3))  # ~9 per cell: same-cell groups and mixed ones
    dense[rng.integers(0, len(dense), size=4)] = np.nan
    import torch

    dense = torch.from_numpy(dense).cuda()  # device input: non-finite positions go through the status flag
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    kw = dict(pipeline=True, status=st, check=False)
    monkeypatch.setenv("SPO_LINE", "0")
    ref = evaluate(dt, "v", dense, **kw).clone()
    for line, vwin in (("1", None), ("2", "1")):
        monkeypatch.setenv("SPO_LINE", line)
        if vwin:
            monkeypatch.setenv("SPO_VWIN", vwin)
        for vg in ("1", "2", "3", "4", "5"):
            monkeypatch.setenv("SPO_VGROUP", vg)
            for knobs in ({}, {"SPO_VDYN": "0"}, {"SPO_VUNI": "0"}, {"SPO_PSPIN": "0"}, {"SPO_VCELL": "0"},
                          {"SPO_VCELL": "1"}, {"SPO_VCELL": "1", "SPO_VDYN": "0"}):
                for k, v in knobs.items():
                    monkeypatch.setenv(k, v)
                got = evaluate(dt, "v", dense, **kw)
                assert _eq(got, ref), (line, vwin, vg, knobs)
                for k in knobs:
                    monkeypatch.delenv(k)

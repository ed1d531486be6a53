"""The k-power table form (spo_b200.h SPO_TABLE_KPOWER, DeviceTable.with_kpower):
z-cubics stored in the power basis, contracted with 7 instead of 12 FMAs per
row group.  Checked here:

* spo_pack_kpower against a numpy restatement of the basis change (bitwise);
* every FAST kernel (generic, per-position TMA, line) on the k-power form
  against the fp64 oracle on random tables (its documented bound, relative
  to the power-basis coefficients, is checked on adversarial tables in
  test_gpu_adversarial.py) -- the k-power form is a different arithmetic,
  so the anchor is the oracle, not the B-spline kernels' bits;
* the three kernels bitwise equal to each other on the k-power form (same FMA
  sequence), across kinds, dtypes, tilings, ragged batches, non-finite
  positions, out_index and lane_limit;
* the contract: STRICT needs the B-spline form, form="kpower" needs with_kpower.
"""
import numpy as np
import pytest

import oracle
from paper_1611_02665_b200 import (ConfigError, ContractError, DeviceTable, DomainError, KernelKind, evaluate,
                                   streams)
from paper_1611_02665_b200.grid import unit_cell_grid

pytestmark = pytest.mark.gpu


def _three(monkeypatch, dt, kind, pos, **kw):
    """(generic, tma, line) outputs on the table's k-power form."""
    outs = [evaluate(dt, kind, pos, pipeline=False, form="kpower", **kw).clone()]
    for v in ("0", "1"):
        monkeypatch.setenv("SPO_LINE", v)
        outs.append(evaluate(dt, kind, pos, pipeline=True, form="kpower", **kw).clone())
    monkeypatch.delenv("SPO_LINE")
    return outs


def _eq(a, b):
    import torch

    return bool(torch.equal(a.nan_to_num(123.0), b.nan_to_num(123.0)))


def _oracle_ok(dt, kind, got, pos, tol, sample):
    names = KernelKind(kind).stream_names
    ref, scale = oracle.eval_f64(kind, dt.reference_soa(), dt.n_splines, dt.grid.spacings, pos[sample])
    s = streams(got, dt, kind)
    g = np.stack([s[n].cpu().numpy()[sample] for n in names], axis=1)
    return oracle.tolerance_check(g, ref, scale, tol)


def _kpower_numpy(data):
    """Restatement of the basis change on a device table's B-spline data
    [m][i'][j'][k'][l] -> [m][i'][j'][4 k0 + r][l] (spo_table.cu kpower_kernel)."""
    c = data.astype(np.float64)
    nz = c.shape[3] - 3
    c0, c1, c2, c3 = (c[:, :, :, r: r + nz] for r in range(4))
    q = np.stack([(c0 + 4.0 * c1 + c2) / 6.0, (c2 - c0) / 2.0, (c0 - 2.0 * c1 + c2) / 2.0,
                  ((c3 - c0) + 3.0 * (c1 - c2)) / 6.0], axis=4)  # [m][i'][j'][k0][r][l]
    return q.reshape(c.shape[:3] + (4 * nz, c.shape[4])).astype(data.dtype)


@pytest.mark.parametrize("f64", [False, True])
def test_pack_kpower_bitwise(f64):
    grid = unit_cell_grid(7)
    dt = (DeviceTable.normal_f64(grid, 40, seed=3, tile_size=16) if f64
          else DeviceTable.random(grid, 70, seed=3, tile_size=32)).with_kpower()
    want = _kpower_numpy(dt.data.cpu().numpy())
    got = dt.kdata.cpu().numpy()
    assert got.shape == want.shape == dt.kpower_shape
    assert np.array_equal(got.view(np.uint8), want.view(np.uint8))


def test_kpower_identity_on_a_cubic():
    """sum_k a_k(t) c_k == q0 + t q1 + t^2 q2 + t^3 q3 for the reference basis
    (grid.py:127-130), exercised through the packed rows of one lane."""
    grid = unit_cell_grid(5)
    dt = DeviceTable.normal_f64(grid, 16, seed=1).with_kpower()
    c = dt.data.cpu().numpy()[0, 2, 3, :, 0]
    q = dt.kdata.cpu().numpy()[0, 2, 3, :, 0].reshape(5, 4)
    for k0 in range(5):
        for t in (0.0, 0.25, 0.5, 0.999):
            s = 1.0 - t
            a = np.array([s ** 3 / 6, (3 * t ** 3 - 6 * t ** 2 + 4) / 6, (-3 * t ** 3 + 3 * t ** 2 + 3 * t + 1) / 6,
                          t ** 3 / 6])
            assert abs(a @ c[k0: k0 + 4] - np.polyval(q[k0][::-1], t)) < 1e-12 * (1 + np.abs(c).max())


@pytest.mark.parametrize("kind", ["v", "vgl", "vgh"])
@pytest.mark.parametrize("tile", ["auto", None])
def test_kpower_fp32_three_kernels_and_oracle(monkeypatch, kind, tile):
    dt = DeviceTable.random(unit_cell_grid(20), 512, seed=5, tile_size=tile).with_kpower()
    pos = np.random.default_rng(2).random((30000 + 17, 3)) * 3.0 - 1.0  # ragged, wrapped inputs
    g, t, ln = _three(monkeypatch, dt, kind, pos)
    assert _eq(g, t) and _eq(g, ln)
    ok, worst = _oracle_ok(dt, kind, ln, pos, 1e-5, np.arange(0, pos.shape[0], 97))
    assert ok, worst


@pytest.mark.parametrize("kind", ["v", "vgl", "vgh"])
def test_kpower_fp64_three_kernels_and_oracle(monkeypatch, kind):
    dt = DeviceTable.normal_f64(unit_cell_grid(16), 128, seed=5).with_kpower()
    pos = np.random.default_rng(3).random((20000, 3))
    g, t, ln = _three(monkeypatch, dt, kind, pos)
    assert _eq(g, t) and _eq(g, ln)
    ok, worst = _oracle_ok(dt, kind, ln, pos, 1e-12, np.arange(0, pos.shape[0], 53))
    assert ok, worst


def test_kpower_close_to_bspline_form():
    dt = DeviceTable.random(unit_cell_grid(24), 256, seed=7).with_kpower()
    pos = np.random.default_rng(4).random((50000, 3))
    a = evaluate(dt, "vgh", pos, form="kpower")
    b = evaluate(dt, "vgh", pos, form="bspline")
    assert a.shape == b.shape
    # not bitwise (different arithmetic), close at fp32 rounding level
    rel = float(((a - b).abs().amax() / b.abs().amax()).item())
    assert 0 < rel < 1e-5


def test_kpower_reference_edge_coordinates(monkeypatch):
    """Cell edges, wrap-around and far-away coordinates (test_grid.py:32-67
    classes) on a non-cubic grid, against the oracle."""
    from paper_1611_02665_b200.grid import GridSpec

    grid = GridSpec(10, 12, 9, 0.1, 1.0 / 12, 1.0 / 9)
    dt = DeviceTable.random(grid, 96, seed=11).with_kpower()
    ax = np.array([0.0, -1e-18, 1.0, 1 - 1e-12, 0.5, 2.7, -0.25, 47.5, 1e6 + 0.3, -3.999999])
    pos = np.stack(np.meshgrid(ax, ax[::-1], np.roll(ax, 3), indexing="ij"), -1).reshape(-1, 3)
    pos = np.concatenate([pos] * 40)  # enough for the pipelined kernels
    g, t, ln = _three(monkeypatch, dt, "vgh", pos)
    assert _eq(g, t) and _eq(g, ln)
    ok, worst = _oracle_ok(dt, "vgh", ln, pos, 1e-5, np.arange(1000))
    assert ok, worst


def test_kpower_nonfinite_out_index_lane_limit(monkeypatch):
    import torch

    dt = DeviceTable.random(unit_cell_grid(16), 256, seed=3).with_kpower()
    P = 6000
    pos = np.random.default_rng(6).random((P, 3))
    pos[[3, 777], [0, 2]] = [np.nan, np.inf]
    dpos = torch.from_numpy(pos).cuda()
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    g, t, ln = _three(monkeypatch, dt, "vgl", dpos, status=st, check=False)
    assert _eq(g, t) and _eq(g, ln) and int(st.item()) == 1
    assert bool(torch.isnan(ln[777]).all()) and not bool(torch.isnan(ln[778]).any())
    with pytest.raises(DomainError):
        evaluate(dt, "vgl", dpos, form="kpower")
    pos[[3, 777], [0, 2]] = 0.5
    perm = torch.from_numpy(np.random.default_rng(8).permutation(P)).cuda()
    outs = []
    for v in ("1", "0"):
        monkeypatch.setenv("SPO_LINE", v)
        o = torch.full((P, 10, dt.lanes), 5.0, device="cuda")
        evaluate(dt, "vgh", pos, o, out_index=perm, pipeline=True, form="kpower")
        buf = torch.full((P, 10, 300), 5.0, device="cuda")
        evaluate(dt, "vgh", pos, buf[:, :, 4:], pipeline=True, lane_limit=201, form="kpower")
        outs.append((o, buf))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    assert bool((outs[0][1][:, :, 205:] == 5.0).all())
    plain = evaluate(dt, "vgh", pos, form="kpower")
    assert torch.equal(outs[0][0][perm], plain)


def test_kpower_contract():
    import ctypes

    from paper_1611_02665_b200 import _abi

    dt = DeviceTable.random(unit_cell_grid(8), 64, seed=1)
    pos = np.random.default_rng(1).random((100, 3))
    with pytest.raises(ContractError):
        evaluate(dt, "vgh", pos, form="kpower")  # no k-power form yet
    dt.with_kpower()
    with pytest.raises(ContractError):
        evaluate(dt, "vgh", pos, mode="strict", form="kpower")
    # strict mode on a table that carries both forms reads the B-spline form
    assert evaluate(dt, "vgh", pos, mode="strict").shape == (100, 10, dt.lanes)
    L = _abi.load()
    g = dt.grid
    rc = L.spo_eval(2, 0, _abi.MODE_STRICT | _abi.TABLE_KPOWER, dt.kdata.data_ptr(), _abi.i32x3(g.counts), dt.nb,
                    dt.n_tiles, _abi.f64x3(g.inverse_spacings), _abi.f64x3(g.spacings), ctypes.c_void_p(0), 0,
                    ctypes.c_void_p(0), 0, 0, None, None, None, 0, None)
    with pytest.raises(ConfigError):
        _abi.check(rc)


def test_kpower_auto_policy():
    """form="auto" reads the B-spline form whatever the table carries and
    however dense the batch: the k-power form's error bound is weaker than
    the north-star one (tests/test_gpu_adversarial.py), so it is opt-in."""
    import torch

    from paper_1611_02665_b200.kernels import eval_form, eval_path

    dt = DeviceTable.random(unit_cell_grid(16), 256, seed=4).with_kpower()
    dense = np.random.default_rng(1).random((2 * 16 ** 3, 3))
    sparse = dense[:600]
    assert eval_path(dt, "vgh", len(dense)) == "window"  # 2 per cell, B-spline form
    assert eval_path(dt, "vgh", len(dense), form="kpower") == "line"
    for p in (dense, sparse):
        assert eval_form(dt, "vgh", len(p)) == "bspline"
        assert eval_form(dt, "vgh", len(p), form="kpower") == "kpower"
        assert torch.equal(evaluate(dt, "vgh", p), evaluate(dt, "vgh", p, form="bspline"))
    assert eval_form(dt, "vgh", len(dense), mode="strict") == "bspline"


def test_kpower_from_host_aos_and_soa():
    """Reference host tables (SoA and AoS layouts, build_table) uploaded, given
    the k-power form: both layouts evaluate bitwise alike on it, within the
    tolerance of the oracle."""
    import torch

    from paper_1611_02665_b200 import FillSpec, build_table
    from paper_1611_02665_b200.grid import GridSpec

    grid = GridSpec(14, 14, 14, 1.0 / 14, 1.0 / 14, 1.0 / 14)
    soa = DeviceTable.from_host(build_table(grid, 96, FillSpec.random(5))).with_kpower()
    aos = DeviceTable.from_host(build_table(grid, 96, FillSpec.random(5), layout="aos")).with_kpower()
    pos = np.random.default_rng(3).random((3 * 14 ** 3, 3))
    a = evaluate(soa, "vgh", pos, form="kpower")
    b = evaluate(aos, "vgh", pos, form="kpower")
    assert torch.equal(a, b)
    ok, worst = _oracle_ok(soa, "vgh", a, pos, 1e-5, np.arange(0, len(pos), 41))
    assert ok, worst


def test_kpower_graph_replay():
    """A CUDA graph of a dense k-power evaluation replays bitwise."""
    import torch

    from paper_1611_02665_b200.graphs import GraphedEvaluator
    from paper_1611_02665_b200.kernels import eval_form

    dt = DeviceTable.random(unit_cell_grid(16), 256, seed=2).with_kpower()
    P = 2 * 16 ** 3
    assert eval_form(dt, "vgh", P, form="kpower") == "kpower"
    ge = GraphedEvaluator(dt, "vgh", P, form="kpower")
    for seed in (1, 2):
        pos = np.random.default_rng(seed).random((P, 3))
        got = ge.run(torch.from_numpy(pos).cuda()).clone()
        assert torch.equal(got, evaluate(dt, "vgh", pos, form="kpower"))


def test_kpower_through_eval_batch():
    """The drop-in eval_batch on a table that carries the k-power form still
    reads the B-spline form (the reference's error contract)."""
    from paper_1611_02665_b200 import WalkerOutputsSoA, collect_streams, eval_batch

    dt = DeviceTable.random(unit_cell_grid(16), 128, seed=6).with_kpower()
    pos = np.random.default_rng(9).random((3 * 16 ** 3 + 5, 3))
    out = WalkerOutputsSoA(128)
    eval_batch(dt, "vgh", pos, out)
    want = streams(evaluate(dt, "vgh", pos[-1:], form="bspline"), dt, "vgh")
    got = collect_streams(out, KernelKind("vgh"))
    for name in KernelKind("vgh").stream_names:
        assert np.array_equal(got[name], want[name].cpu().numpy()[0]), name

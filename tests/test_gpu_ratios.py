"""Fused consumer epilogue (evaluate_ratios): the per-position contraction of
every output stream with a coefficient row equals the same contraction of
evaluate()'s outputs, for fp32 and fp64 tables, tiled and not; deterministic."""
import numpy as np
import pytest

from paper_1611_02665_b200 import ConfigError, DeviceTable, DomainError, evaluate, evaluate_ratios, streams
from paper_1611_02665_b200.grid import GridSpec, unit_cell_grid
from paper_1611_02665_b200.kernels import KernelKind

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t

    assert t.cuda.is_available()
    return t


def reference_ratios(torch, dt, kind, pos, coef):
    out = evaluate(dt, kind, pos, pipeline=True)
    s = streams(out, dt, kind)
    names = KernelKind(kind).stream_names
    full = torch.stack([s[k].double() for k in names], dim=1)  # [P][S][N]
    return torch.einsum("psn,pn->ps", full, coef.double())


@pytest.mark.parametrize("kind", ["v", "vgl", "vgh"])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_ratios_match_contracted_outputs(torch, kind, dtype):
    grid = unit_cell_grid(20)
    rng = np.random.default_rng(5)
    if dtype == "f32":
        dt = DeviceTable.random(grid, 300, seed=2, tile_size=128)
        tdt = torch.float32
        rtol = 1e-6
    else:
        dt = DeviceTable.normal_f64(grid, 200, seed=2, tile_size=64)
        tdt = torch.float64
        rtol = 1e-12
    pos = rng.random((5000, 3)) * 2.0 - 0.5
    coef = torch.from_numpy(rng.standard_normal((5000, dt.n_splines))).to("cuda", tdt)
    got = evaluate_ratios(dt, kind, pos, coef)
    want = reference_ratios(torch, dt, kind, pos, coef)
    scale = want.abs().max()
    assert float((got - want).abs().max() / scale) < rtol
    again = evaluate_ratios(dt, kind, pos, coef)
    assert torch.equal(got, again)  # fixed-order reduction: bitwise reproducible


def test_ratios_untiled_and_errors(torch):
    grid = GridSpec(12, 13, 14, 0.1, 0.2, 0.3)
    dt = DeviceTable.random(grid, 256, seed=1, tile_size=None)  # 1 KB rows: two 512-byte chunks
    pos = np.random.default_rng(1).random((777, 3)) * 3.0
    coef = torch.ones((777, 256), dtype=torch.float32, device="cuda")
    got = evaluate_ratios(dt, "vgh", pos, coef)
    want = reference_ratios(torch, dt, "vgh", pos, coef)
    assert float((got - want).abs().max() / want.abs().max()) < 1e-6
    odd = DeviceTable.random(grid, 96, seed=1, tile_size=None)  # 384-byte rows
    with pytest.raises(ConfigError):
        evaluate_ratios(odd, "v", pos, torch.ones((777, 96), device="cuda"))
    bad = pos.copy()
    bad[3, 0] = np.nan
    with pytest.raises(DomainError):
        evaluate_ratios(dt, "v", bad, coef)


@pytest.mark.parametrize("kind,dtype", [("vgh", "f32"), ("vgl", "f32"), ("vgh", "f64")])
def test_ratios_line_path(torch, monkeypatch, kind, dtype):
    """Dense batches run the line-window kernel's ratio epilogue: bitwise equal
    to the per-position kernel's (same lane dots, same warp reduction, same
    fixed-order unit sum) and to the contraction of evaluate()'s outputs."""
    grid = unit_cell_grid(16)
    rng = np.random.default_rng(8)
    if dtype == "f32":
        dt = DeviceTable.random(grid, 256, seed=3)
        tdt, rtol = torch.float32, 1e-6
    else:
        dt = DeviceTable.normal_f64(grid, 128, seed=3)
        tdt, rtol = torch.float64, 1e-12
    P = 12000  # ~3 positions per cell
    pos = rng.random((P, 3))
    pos[17] = np.nan
    coef = torch.from_numpy(rng.standard_normal((P, dt.n_splines))).to("cuda", tdt)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    monkeypatch.setenv("SPO_LINE", "1")
    a = evaluate_ratios(dt, kind, torch.from_numpy(pos).cuda(), coef, status=st, check=False)
    monkeypatch.setenv("SPO_LINE", "0")
    b = evaluate_ratios(dt, kind, torch.from_numpy(pos).cuda(), coef, check=False)
    assert torch.equal(a.nan_to_num(7.0), b.nan_to_num(7.0)) and int(st.item()) == 1
    assert bool(torch.isnan(a[17]).all())
    ok = torch.ones(P, dtype=torch.bool)
    ok[17] = False
    monkeypatch.delenv("SPO_LINE")
    want = reference_ratios(torch, dt, kind, pos[ok.numpy()], coef[ok.cuda()])
    assert float((a[ok.cuda()] - want).abs().max() / want.abs().max()) < rtol


@pytest.mark.parametrize("per_cell", [3, 10])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_ratios_v_position_groups(torch, monkeypatch, dtype, per_cell):
    """V on dense batches: the ratio epilogue inside the line kernel's V position
    groups (fixed groups at 3 per cell, groups aligned to cells at 10 per cell,
    both forced too): bitwise equal to the per-position kernel's ratios, NaN
    rows for non-finite positions, and equal to the contracted outputs."""
    grid = unit_cell_grid(12)
    rng = np.random.default_rng(21)
    if dtype == "f32":
        dt = DeviceTable.random(grid, 300, seed=3, tile_size=128)
        tdt, rtol = torch.float32, 1e-6
    else:
        dt = DeviceTable.normal_f64(grid, 144, seed=3, tile_size=64)
        tdt, rtol = torch.float64, 1e-12
    P = per_cell * 12 ** 3 + 37
    pos = rng.random((P, 3)) * 2.0 - 0.5
    pos[[5, P - 1]] = np.nan
    dpos = torch.from_numpy(pos).cuda()
    coef = torch.from_numpy(rng.standard_normal((P, dt.n_splines))).to("cuda", tdt)
    monkeypatch.setenv("SPO_LINE", "0")
    ref = evaluate_ratios(dt, "v", dpos, coef, check=False)
    monkeypatch.setenv("SPO_LINE", "1")
    for knobs in ({}, {"SPO_VCELL": "0"}, {"SPO_VCELL": "1"}, {"SPO_VGROUP": "1"}, {"SPO_VGROUP": "4", "SPO_VCELL": "1"}):
        for k, v in knobs.items():
            monkeypatch.setenv(k, v)
        got = evaluate_ratios(dt, "v", dpos, coef, check=False)
        for k in knobs:
            monkeypatch.delenv(k)
        assert torch.equal(got.nan_to_num(7.0), ref.nan_to_num(7.0)), knobs
        assert bool(torch.isnan(got[5]).all()) and bool(torch.isnan(got[P - 1]).all())
    monkeypatch.delenv("SPO_LINE")
    ok = np.ones(P, bool)
    ok[[5, P - 1]] = False
    want = reference_ratios(torch, dt, "v", pos[ok], coef[torch.from_numpy(ok).cuda()])
    assert float((ref[torch.from_numpy(ok).cuda()] - want).abs().max() / want.abs().max()) < rtol


@pytest.mark.parametrize("line", ["0", "1"])
@pytest.mark.parametrize("kind", ["v", "vgl", "vgh"])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_ratios_against_oracle(torch, monkeypatch, kind, dtype, line):
    """Anchored on the f64 oracle: want[p, s] = sum_n
    oracle(p, s, n) * coef[p, n] in fp64.  Bound: the north-star per-element
    bound carried through the contraction, tol * sum_n sum|w*c|(p, s, n) *
    |coef[p, n]|, with tol doubled for the lane dots' own rounding (fp32
    products summed within 128-orbital chunks, fp64 across chunks)."""
    import oracle

    grid = unit_cell_grid(16)
    rng = np.random.default_rng(12)
    if dtype == "f32":
        dt = DeviceTable.random(grid, 512, seed=9)
        tdt, tol = torch.float32, 2e-5
    else:
        dt = DeviceTable.normal_f64(grid, 256, seed=9)
        tdt, tol = torch.float64, 2e-12
    P = 3 * 16 ** 3  # dense: the line path when SPO_LINE=1
    pos = rng.random((P, 3)) * 2.0 - 0.5
    coef_np = rng.standard_normal((P, dt.n_splines))
    coef = torch.from_numpy(coef_np).to("cuda", tdt)
    monkeypatch.setenv("SPO_LINE", line)
    got = evaluate_ratios(dt, kind, pos, coef).cpu().numpy()
    monkeypatch.delenv("SPO_LINE")
    sel = np.arange(0, P, 7)
    ref, scale = oracle.eval_f64(kind, dt.reference_soa(), dt.n_splines, grid.spacings, pos[sel])
    c = coef.double().cpu().numpy()[sel]  # the coefficients as the kernel saw them
    want = np.einsum("psn,pn->ps", ref, c)
    bound = tol * np.einsum("psn,pn->ps", scale, np.abs(c))
    err = np.abs(got[sel] - want)
    assert (err <= bound).all(), float((err / bound).max())


@pytest.mark.parametrize("kind", ["v", "vgh"])
def test_orbital_sharded_ratios_sum_to_the_full_table(torch, kind):
    """multi.evaluate_ratios_orbital_sharded, the slices of a 3-way orbital
    partition evaluated one after the other on this GPU (world 1: the reduce is
    the identity): the partials add up to evaluate_ratios on the full table,
    which is anchored on the f64 oracle (test_ratios_against_oracle*)."""
    from paper_1611_02665_b200.multi import (OrbitalPartition, evaluate_ratios_orbital_sharded,
                                             shard_table_for_rank)

    grid = unit_cell_grid(16)
    rng = np.random.default_rng(9)
    dt = DeviceTable.normal_f64(grid, 208, seed=4)
    pos = rng.random((3000, 3)) * 2.0 - 0.5
    coef = torch.from_numpy(rng.standard_normal((3000, 208))).cuda()
    want = evaluate_ratios(dt, kind, pos, coef)
    part = OrbitalPartition.make(208, 3, quantum=16)
    total = torch.zeros_like(want)
    for r in range(3):
        lo, hi = part.local(r)
        local = shard_table_for_rank(dt, part, r, tile_size=64)  # the epilogue needs 512-byte rows
        total += evaluate_ratios_orbital_sharded(local, kind, pos, coef[:, lo:hi].contiguous())
    assert float((total - want).abs().max() / want.abs().max()) < 1e-12  # fp64 partial sums, another order

"""GPU parity: the CUDA path through the C ABI against the oracle and the
reference's golden vectors.  Bars: stencil indices / fp32 weights bit-exact;
fast mode within 1e-5 * sum|w*c| per element (fp32) and 1e-12 (fp64);
strict mode bitwise equal to the reference fp32 kernels."""
import hashlib

import numpy as np
import pytest

import oracle
from paper_1611_02665_b200 import _abi
from paper_1611_02665_b200.coeffs import FillSpec, build_table, tile_table
from paper_1611_02665_b200.device import DeviceTable
from paper_1611_02665_b200.grid import GridSpec, unit_cell_grid
from paper_1611_02665_b200.kernels import KernelKind, evaluate, streams

pytestmark = pytest.mark.gpu

KINDS = ("v", "vgl", "vgh")
TOL32 = 1e-5   # north_star fp32 tolerance, scaled by sum|w*c|
TOL64 = 1e-12  # north_star fp64 tolerance


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def torch():
    import torch as t

    assert t.cuda.is_available()
    return t


@pytest.fixture(scope="module")
def cfg1(torch):
    host = build_table(unit_cell_grid(16), 64, FillSpec.random(0))
    return host, DeviceTable.from_host(host)


def run(dt, kind, pos, mode="fast", pipeline="auto"):
    out = evaluate(dt, kind, pos, mode=mode, pipeline=pipeline)
    s = streams(out, dt, kind)
    names = KernelKind(kind).stream_names
    return np.stack([s[k].cpu().numpy() for k in names], axis=1)


# ------------------------------------------------------------ prologue --

def test_prologue_bit_exact(torch, golden_mapping):
    g = golden_mapping
    L = _abi.load()
    dev = torch.device("cuda")
    xs = g["xs"]
    for a, (dinv, cnt) in enumerate(g["pairs"]):
        n = int(cnt)
        pos = torch.from_numpy(np.stack([xs, xs, xs], axis=1).copy()).to(dev)
        idx = torch.empty((xs.size, 3), dtype=torch.int32, device=dev)
        t = torch.empty((xs.size, 3), dtype=torch.float64, device=dev)
        _abi.check(L.spo_prologue(0, _abi.i32x3((n, n, n)), _abi.f64x3((dinv,) * 3),
                                  _abi.f64x3((1.0 / dinv,) * 3), pos.data_ptr(), xs.size,
                                  idx.data_ptr(), t.data_ptr(), None, None))
        torch.cuda.synchronize()
        np.testing.assert_array_equal(idx[:, 0].cpu().numpy(), g["i0"][a])
        np.testing.assert_array_equal(t[:, 0].cpu().numpy(), g["t"][a])


def test_basis_weights_bit_exact(torch, golden_mapping):
    g = golden_mapping
    L = _abi.load()
    t = torch.from_numpy(g["ts"]).cuda()
    for a, dinv in enumerate(g["dinvs"]):
        w = torch.empty((t.numel(), 3, 4), dtype=torch.float32, device="cuda")
        _abi.check(L.spo_basis_weights(0, t.data_ptr(), t.numel(), float(dinv), 1.0 / dinv, w.data_ptr(), None))
        np.testing.assert_array_equal(w.cpu().numpy(), g["w32"][a])
        w64 = torch.empty((t.numel(), 3, 4), dtype=torch.float64, device="cuda")
        _abi.check(L.spo_basis_weights(1, t.data_ptr(), t.numel(), float(dinv), 1.0 / dinv, w64.data_ptr(), None))
        np.testing.assert_allclose(w64.cpu().numpy(), g["w64"][a], rtol=4e-16, atol=4e-16 * dinv * dinv)


# -------------------------------------------------------------- tables --

def test_device_fill_equals_reference_table(torch, cfg1, golden_cfg1):
    dt = DeviceTable.random(unit_cell_grid(16), 64, seed=0)
    assert sha(dt.reference_soa()) == str(golden_cfg1["table_sha"])
    assert torch.equal(dt.data, cfg1[1].data)
    # wrap ring: padded row i'=0 equals grid row nx-1, i'=nx+1 equals row 0
    d = dt.data[0]
    assert torch.equal(d[0, 1:17, 1:17], d[16, 1:17, 1:17])
    assert torch.equal(d[17, 1:17, 1:17], d[1, 1:17, 1:17])
    assert torch.equal(d[1:17, 1:17, 18], d[1:17, 1:17, 2])


def test_device_fill_tiled_and_ragged(torch, golden_small):
    for tag in ("ragged5", "g12n24", "g5x4x6n7", "g8n33"):
        meta = golden_small[f"{tag}_meta"]
        counts, n, seed = tuple(int(x) for x in meta[:3]), int(meta[3]), int(meta[4])
        spac = tuple(float(x) for x in golden_small[f"{tag}_spacing"])
        grid = GridSpec(*counts, *spac)
        for ts in (None, 4, 7):
            dt = DeviceTable.random(grid, n, seed=seed, tile_size=ts)
            assert sha(dt.reference_soa()) == str(golden_small[f"{tag}_table_sha"]), (tag, ts)


# -------------------------------------------------------------- config 1 --

@pytest.mark.parametrize("pipeline", [True, False])
@pytest.mark.parametrize("kind", KINDS)
def test_cfg1_fast_within_tolerance(cfg1, golden_cfg1, kind, pipeline):
    host, dt = cfg1
    pos = golden_cfg1["positions"]
    got = run(dt, kind, pos, pipeline=pipeline)
    ref, scale = oracle.eval_f64(kind, host.data, 64, host.grid.spacings, pos)
    ok, worst = oracle.tolerance_check(got, ref, scale, TOL32)
    assert ok, worst
    np.testing.assert_allclose(got[:24], golden_cfg1[f"{kind}_f64_head"], rtol=0, atol=1e-5 * np.abs(scale[:24]).max())


@pytest.mark.parametrize("kind", KINDS)
def test_cfg1_strict_bitwise_all_positions(cfg1, golden_cfg1, kind):
    """Strict mode == the reference numba fp32 kernels on all 512 x S x 64 outputs."""
    _, dt = cfg1
    got = run(dt, kind, golden_cfg1["positions"], mode="strict")
    np.testing.assert_array_equal(got[:64], golden_cfg1[f"{kind}_f32_head"])
    assert sha(got) == str(golden_cfg1[f"{kind}_f32_sha"])
    edge = run(dt, kind, golden_cfg1["edge_positions"], mode="strict")
    np.testing.assert_array_equal(edge, golden_cfg1[f"{kind}_f32_edge"])


@pytest.mark.parametrize("tile", [16, 24, 32, 5])
def test_cfg1_tiled_bitwise_equal_untiled(cfg1, golden_cfg1, tile):
    host, dt = cfg1
    tiled = DeviceTable.from_host(host, tile_size=tile)
    assert tiled.n_tiles == -(-64 // tile)
    pos = golden_cfg1["positions"]
    for mode in ("fast", "strict"):
        np.testing.assert_array_equal(run(tiled, "vgh", pos, mode), run(dt, "vgh", pos, mode))
    assert sha(run(tiled, "vgh", pos, "strict")) == str(golden_cfg1["vgh_f32_tiled_sha"])


def test_reference_tiled_table_upload(cfg1, golden_cfg1):
    host, dt = cfg1
    tiled_host = tile_table(host, 16)
    tdt = DeviceTable.from_host(tiled_host)
    assert tdt.n_tiles == 4 and tdt.nb == 32
    np.testing.assert_array_equal(run(tdt, "vgh", golden_cfg1["positions"][:32], "strict"),
                                  golden_cfg1["vgh_f32_head"][:32])


def test_value_stream_identical_across_kinds(cfg1, golden_cfg1):
    _, dt = cfg1
    pos = golden_cfg1["positions"]
    for mode in ("fast", "strict"):
        v = run(dt, "v", pos, mode)[:, 0]
        vgl = run(dt, "vgl", pos, mode)
        vgh = run(dt, "vgh", pos, mode)
        np.testing.assert_array_equal(v, vgl[:, 0])
        np.testing.assert_array_equal(v, vgh[:, 0])
        np.testing.assert_array_equal(vgl[:, 1:4], vgh[:, 1:4])


@pytest.mark.parametrize("kind", KINDS)
def test_pipelined_and_generic_kernels_bitwise_equal(cfg1, golden_cfg1, kind):
    """The TMA-pipelined and the generic fast kernels run the same FMA
    sequence per lane: identical bits, tiled or not."""
    host, dt = cfg1
    pos = golden_cfg1["positions"]
    for table in (dt, DeviceTable.from_host(host, tile_size=32)):
        a = evaluate(table, kind, pos, pipeline=True)
        b = evaluate(table, kind, pos, pipeline=False)
        assert bool((a == b).all())


def test_laplacian_is_hessian_trace(cfg1, golden_cfg1):
    _, dt = cfg1
    pos = golden_cfg1["positions"]
    vgl = run(dt, "vgl", pos)
    vgh = run(dt, "vgh", pos).astype(np.float64)
    trace = vgh[:, 4] + vgh[:, 7] + vgh[:, 9]
    assert np.abs(vgl[:, 4] - trace).max() / np.abs(trace).max() <= 1e-4


def test_padding_lanes_are_zero(torch):
    host = build_table(GridSpec(12, 12, 12), 5, FillSpec.random(4))
    dt = DeviceTable.from_host(host)
    out = evaluate(dt, "vgh", np.array([[2.2, 3.3, 4.4], [1.0, 2.0, 3.0]]))
    assert out.shape == (2, 10, 32)
    assert (out[:, :, 5:] == 0).all()


@pytest.mark.parametrize("tag", ["ragged5", "g12n24", "g5x4x6n7", "g8n33"])
def test_small_cases(torch, golden_small, tag):
    meta = golden_small[f"{tag}_meta"]
    counts, n, seed = tuple(int(x) for x in meta[:3]), int(meta[3]), int(meta[4])
    spac = tuple(float(x) for x in golden_small[f"{tag}_spacing"])
    host = build_table(GridSpec(*counts, *spac), n, FillSpec.random(seed))
    dt = DeviceTable.from_host(host)
    pos = golden_small[f"{tag}_positions"]
    for kind in KINDS:
        np.testing.assert_array_equal(run(dt, kind, pos, "strict"), golden_small[f"{tag}_{kind}_f32"])
        ref, scale = oracle.eval_f64(kind, host.data, n, spac, pos)
        for pipeline in (True, False):
            ok, worst = oracle.tolerance_check(run(dt, kind, pos, pipeline=pipeline), ref, scale, TOL32)
            assert ok, (kind, pipeline, worst)


def test_out_index_scatter_is_bitwise(torch, cfg1, golden_cfg1):
    _, dt = cfg1
    pos = golden_cfg1["positions"]
    perm = np.random.default_rng(5).permutation(pos.shape[0])
    base = evaluate(dt, "vgh", pos)
    out = torch.empty_like(base)
    idx = torch.from_numpy(perm.astype(np.int64)).cuda()
    evaluate(dt, "vgh", pos[perm], out, out_index=idx)  # out[perm[q]] = eval(pos[perm[q]])
    assert torch.equal(out, base)


def test_nonfinite_positions_raise(torch, cfg1):
    from paper_1611_02665_b200.errors import DomainError

    _, dt = cfg1
    with pytest.raises(DomainError):
        evaluate(dt, "v", np.array([[0.1, 0.2, 0.3], [np.nan, 0.0, 0.0]]))
    dpos = torch.tensor([[0.1, 0.2, 0.3], [0.0, np.inf, 0.0]], dtype=torch.float64, device="cuda")
    with pytest.raises(DomainError):
        evaluate(dt, "vgh", dpos)
    for pipeline in (True, False):
        with pytest.raises(DomainError):
            evaluate(dt, "vgh", dpos, pipeline=pipeline)
        status = torch.zeros(1, dtype=torch.int32, device="cuda")
        out = evaluate(dt, "vgh", dpos, status=status, check=False, pipeline=pipeline)
        assert int(status.item()) == 1
        assert torch.isnan(out[1]).all() and torch.isfinite(out[0]).all()


# ---------------------------------------------------------------- fp64 --

@pytest.mark.parametrize("kind", KINDS)
def test_fp64_within_1e12(torch, kind):
    grid = unit_cell_grid(12)
    dt = DeviceTable.normal_f64(grid, 40, seed=3)
    host = dt.reference_soa()
    assert host.dtype == np.float64
    pos = np.random.default_rng(9).random((200, 3)) * 3.0 - 1.0
    got = run(dt, kind, pos)
    ref, scale = oracle.eval_f64(kind, host, 40, grid.spacings, pos)
    ok, worst = oracle.tolerance_check(got, ref, scale, TOL64)
    assert ok, worst
    tiled = DeviceTable.normal_f64(grid, 40, seed=3, tile_size=16)
    np.testing.assert_array_equal(run(tiled, kind, pos), got)
    # the fp64 TMA-pipelined kernel runs the generic kernel's DFMA sequence
    for table in (dt, tiled, DeviceTable.normal_f64(grid, 40, seed=3, tile_size=32)):
        np.testing.assert_array_equal(run(table, kind, pos, pipeline=True), got)


def test_fp64_normal_fill_moments(torch):
    dt = DeviceTable.normal_f64(unit_cell_grid(16), 64, seed=0)
    v = dt.reference_soa()[..., :64].reshape(-1)
    assert abs(v.mean()) < 0.01 and abs(v.std() - 1.0) < 0.01


# ------------------------------------------------------- edge cases --

def test_pipelined_edge_cases(torch, golden_mapping):
    """The TMA path on awkward inputs: huge / negative / boundary coordinates,
    a ragged tiled table (tile 24 -> 32-lane rows), strided output views,
    out_index scatter, P = 1 and P = 0, two streams at once."""
    grid = GridSpec(20, 24, 28, 0.05, 1 / 24, 1 / 28)
    host = build_table(grid, 72, FillSpec.random(11))
    xs = golden_mapping["xs"]
    rng = np.random.default_rng(3)
    pos = np.stack([rng.choice(xs, 3000), rng.choice(xs, 3000), rng.random(3000)], axis=1)
    ref_dt = DeviceTable.from_host(host, tile_size=None)
    base = evaluate(ref_dt, "vgh", pos, pipeline=False)
    for tile in (None, 24, 32):
        dt = DeviceTable.from_host(host, tile_size=tile)
        got = streams(evaluate(dt, "vgh", pos, pipeline=True), dt, "vgh")
        want = streams(base, ref_dt, "vgh")
        for k in want:
            assert torch.equal(got[k], want[k]), (tile, k)
    ref, scale = oracle.eval_f64("vgh", host.data, 72, grid.spacings, pos[:200])
    ok, worst = oracle.tolerance_check(run(ref_dt, "vgh", pos[:200], pipeline=True), ref, scale, TOL32)
    assert ok, worst
    # strided output view + out_index scatter
    big = torch.zeros((3000, 10, 256), dtype=torch.float32, device="cuda")
    view = big[:, :, 64:64 + ref_dt.lanes]
    perm = rng.permutation(3000)
    evaluate(ref_dt, "vgh", pos[perm], view, out_index=torch.from_numpy(perm).cuda(), pipeline=True)
    assert torch.equal(view, base) and (big[:, :, :64] == 0).all()
    # tiny and empty batches
    one = evaluate(ref_dt, "vgh", pos[:1], pipeline=True)
    assert torch.equal(one[0], base[0])
    empty = evaluate(ref_dt, "vgh", np.zeros((0, 3)), pipeline=True)
    assert empty.shape[0] == 0
    # two streams concurrently (separate workspaces and tickets)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(s1):
        a = evaluate(ref_dt, "vgh", pos, pipeline=True, check=False)
    with torch.cuda.stream(s2):
        b = evaluate(ref_dt, "vgl", pos, pipeline=True, check=False)
    torch.cuda.synchronize()
    assert torch.equal(a, base)
    assert torch.equal(b[:, :4], base[:, :4])


def test_abi_rejects_host_pointers(torch, cfg1):
    """A host pointer where device memory is expected is a ContractError, not
    a kernel fault."""
    import ctypes

    _, dt = cfg1
    L = _abi.load()
    pos = torch.zeros((4, 3), dtype=torch.float64, device="cuda")
    out = torch.empty((4, 1, dt.lanes), dtype=torch.float32, device="cuda")
    host_table = np.zeros(dt.data.numel(), dtype=np.float32)
    g = dt.grid
    rc = L.spo_eval(0, 0, 0, host_table.ctypes.data, _abi.i32x3(g.counts), dt.nb, dt.n_tiles,
                    _abi.f64x3(g.inverse_spacings), _abi.f64x3(g.spacings), pos.data_ptr(), 4,
                    out.data_ptr(), dt.lanes, dt.lanes, None, None, None, 0, ctypes.c_void_p(0))
    assert rc == 1 and b"table" in L.spo_last_error()
    host_pos = np.zeros((4, 3))
    rc = L.spo_eval(0, 0, 0, dt.data.data_ptr(), _abi.i32x3(g.counts), dt.nb, dt.n_tiles,
                    _abi.f64x3(g.inverse_spacings), _abi.f64x3(g.spacings), host_pos.ctypes.data, 4,
                    out.data_ptr(), dt.lanes, dt.lanes, None, None, None, 0, ctypes.c_void_p(0))
    assert rc == 1 and b"positions" in L.spo_last_error()

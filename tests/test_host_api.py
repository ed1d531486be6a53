"""Host-side mirror of the reference API (no GPU): grid spec, tables, fills,
tiling, output buffers, argument validation that happens before
any device call.  Mirrors pkg/tests/test_grid.py / test_coeffs.py."""
import numpy as np
import pytest

from paper_1611_02665_b200 import (
    CoeffTableAoS,
    CoeffTableSoA,
    ConfigError,
    ContractError,
    DomainError,
    FillSpec,
    GridSpec,
    KernelKind,
    WalkerOutputsAoS,
    WalkerOutputsSoA,
    allocate_outputs,
    build_table,
    collect_streams,
    convert_aos_to_soa,
    eval_batch,
    eval_tiled,
    eval_v,
    padded_count,
    tile_table,
)
from paper_1611_02665_b200.coeffs import aligned_zeros
from paper_1611_02665_b200.kernels import as_kind
from paper_1611_02665_b200.workloads import bytes_per_position


def test_gridspec_validation():
    with pytest.raises(ConfigError):
        GridSpec(3, 48, 48)
    with pytest.raises(ConfigError):
        GridSpec(48, 48, 48, dx=0.0)
    with pytest.raises(ConfigError):
        GridSpec(48, 48, 48, periodic=False)
    g = GridSpec(48, 48, 60, dx=0.5)
    assert g.lengths == (24.0, 48.0, 60.0)
    assert g.n_points == 48 * 48 * 60
    assert g.padded_counts == (51, 51, 63)
    assert GridSpec(64, 64, 64, 1 / 64, 1 / 64, 1 / 64).inverse_spacings == (64.0, 64.0, 64.0)


def test_padded_count_and_alignment():
    assert [padded_count(n) for n in (1, 16, 17, 64, 4096)] == [16, 16, 32, 64, 4096]
    for shape in ((7,), (3, 5), (4, 4, 4, 16)):
        a = aligned_zeros(shape)
        assert a.ctypes.data % 64 == 0 and a.shape == shape


def test_fills_and_determinism():
    g = GridSpec(8, 8, 8)
    a = build_table(g, 5, FillSpec.random(3))
    b = build_table(g, 5, FillSpec.random(3))
    np.testing.assert_array_equal(a.data, b.data)
    assert (a.data[..., 5:] == 0).all()
    assert a.data[..., :5].min() >= -1.0 and a.data[..., :5].max() < 1.0
    c = build_table(g, 4, FillSpec.constant(2.5))
    assert (c.data[..., :4] == 2.5).all()
    lin = build_table(g, 2, FillSpec.linear_index("y"))
    assert lin.data[1, 3, 5, 0] == 3.0
    with pytest.raises(ConfigError):
        FillSpec("gauss")
    with pytest.raises(ConfigError):
        build_table(g, 0, FillSpec.constant(1))


def test_layout_transforms_round_trip():
    g = GridSpec(5, 4, 6)
    aos = build_table(g, 7, FillSpec.random(1), layout="aos")
    soa = convert_aos_to_soa(aos)
    np.testing.assert_array_equal(np.moveaxis(aos.data, 0, -1), soa.data[..., :7])
    soa2 = build_table(g, 7, FillSpec.random(1))
    np.testing.assert_array_equal(soa.data, soa2.data)
    tiled = tile_table(soa, 7)
    assert tiled.n_tiles == 1
    with pytest.raises(ConfigError):
        tile_table(soa, 3)
    with pytest.raises(ContractError):
        tile_table(aos, 7)


def test_tiling_conserves_elements():
    soa = build_table(GridSpec(6, 6, 6), 24, FillSpec.random(2))
    tiled = tile_table(soa, 8)
    cat = np.concatenate([t.data[..., :8] for t in tiled.tiles], axis=-1)
    np.testing.assert_array_equal(cat, soa.data[..., :24])
    assert tiled.nbytes == 3 * 6 ** 3 * 16 * 4


def test_footprint_known_answer():
    # test_coeffs.py:149-154: 48^3 grid, N=128 -> 56,623,104 bytes
    assert 48 ** 3 * padded_count(128) * 4 == 56623104


def test_tables_are_immutable():
    soa = build_table(GridSpec(4, 4, 4), 3, FillSpec.random(0))
    with pytest.raises(ValueError):
        soa.data[0, 0, 0, 0] = 1.0
    with pytest.raises(ContractError):
        CoeffTableSoA(GridSpec(4, 4, 4), 3, np.zeros((4, 4, 4, 3), np.float32))
    with pytest.raises(ContractError):
        CoeffTableAoS(GridSpec(4, 4, 4), np.zeros((2, 4, 4, 5), np.float32))


def test_output_buffers():
    out = WalkerOutputsSoA(20)
    assert out.n_padded == 32 and out.g.shape == (3, 32) and out.h.shape == (6, 32)
    assert set(out.streams(KernelKind.VGL)) == {"v", "gx", "gy", "gz", "l"}
    aos = WalkerOutputsAoS(3)
    block = np.arange(30, dtype=np.float32).reshape(10, 3)
    aos.store(KernelKind.VGH, block)
    h = aos.h.reshape(3, 3, 3)
    np.testing.assert_array_equal(h, np.swapaxes(h, 1, 2))
    s = aos.streams(KernelKind.VGH)
    np.testing.assert_array_equal(s["hyz"], block[8])
    t = tile_table(build_table(GridSpec(4, 4, 4), 8, FillSpec.random(0)), 4)
    outs = allocate_outputs(t)
    assert len(outs) == 2
    assert collect_streams(outs, "v")["v"].shape == (8,)


def test_kind_aliases():
    assert as_kind("VGH") is KernelKind.VGH
    assert KernelKind.VGH.stream_names[4:] == ("hxx", "hxy", "hxz", "hyy", "hyz", "hzz")
    assert KernelKind.VGH.output_streams("aos") == 13
    with pytest.raises(ContractError):
        as_kind("vg")


def test_validation_before_device_calls():
    soa = build_table(GridSpec(4, 4, 4), 3, FillSpec.random(0))
    out = allocate_outputs(soa)
    with pytest.raises(DomainError):
        eval_v(soa, (np.nan, 0, 0), out)
    with pytest.raises(ContractError):
        eval_v(soa, (0, 0, 0), WalkerOutputsAoS(3))
    with pytest.raises(ContractError):
        eval_batch(soa, "v", np.zeros((2, 4)), out)
    with pytest.raises(ContractError):
        eval_tiled(soa, "v", (0, 0, 0), [out])


def test_roofline_bytes_model():
    # 64*Npad*4 + S*Npad*4 per position
    assert bytes_per_position("vgh", 4096) == 1212416
    assert bytes_per_position("vgl", 2048) == 565248
    assert bytes_per_position("v", 512) == 133120
    assert bytes_per_position("vgh", 64) == 18944

"""Pin the CPU oracle (both restatements) against fixtures generated from the
reference itself (tests/golden/make_golden.py).  CPU only."""
import hashlib

import numpy as np
import pytest

import oracle
from paper_1611_02665_b200.coeffs import FillSpec, build_table
from paper_1611_02665_b200.grid import GridSpec, unit_cell_grid

KINDS = ("v", "vgl", "vgh")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_numpy_map_axis_bitwise(golden_mapping):
    g = golden_mapping
    for a, (dinv, cnt) in enumerate(g["pairs"]):
        i0, t = oracle.map_axis(g["xs"], dinv, cnt)
        np.testing.assert_array_equal(i0, g["i0"][a])
        np.testing.assert_array_equal(t, g["t"][a])


def test_c_map_axis_bitwise(golden_mapping):
    g = golden_mapping
    for a, (dinv, cnt) in enumerate(g["pairs"]):
        for b in range(0, g["xs"].size, 7):
            i0, t = oracle.c_map_axis(g["xs"][b], dinv, cnt)
            assert i0 == g["i0"][a, b]
            assert t == g["t"][a, b] or (np.isnan(t) and np.isnan(g["t"][a, b]))


def test_mapping_known_answers():
    # test_grid.py:32-50 (dx = 1, n = 48)
    i0, t = oracle.map_axis(np.array([2.7, 47.5, -0.25]), 1.0, 48.0)
    assert i0.tolist() == [2, 47, 47]
    assert t[1] == 0.5 and t[2] == 0.75
    assert oracle.c_map_axis(-1e-18, 48.0, 48.0) == (0, 0.0)
    assert oracle.c_map_axis(1.0, 48.0, 48.0) == (0, 0.0)


def test_weights_f32_bitwise(golden_mapping):
    g = golden_mapping
    for a, dinv in enumerate(g["dinvs"]):
        np.testing.assert_array_equal(oracle.weights_f32(g["ts"], dinv), g["w32"][a])
        for b in range(0, g["ts"].size, 11):
            np.testing.assert_array_equal(oracle.c_weights_f32(g["ts"][b], dinv), g["w32"][a, b])


def test_weights_f64_bitwise(golden_mapping):
    g = golden_mapping
    for a, dinv in enumerate(g["dinvs"]):
        for b in range(0, g["ts"].size, 5):
            t = float(g["ts"][b])
            np.testing.assert_array_equal(oracle.weights_f64(t, 1.0 / dinv), g["w64"][a, b])
            np.testing.assert_array_equal(oracle.c_weights_f64(t, 1.0 / dinv), g["w64"][a, b])


def test_weight_known_answers():
    # test_grid.py:70-83
    w = oracle.weights_f32(0.0, 1.0)
    np.testing.assert_array_equal(w[1], np.float32([-0.5, 0.0, 0.5, 0.0]))
    np.testing.assert_array_equal(w[2], np.float32([1.0, -2.0, 1.0, 0.0]))
    np.testing.assert_allclose(oracle.weights_f32(0.5, 1.0)[0], [1 / 48, 23 / 48, 23 / 48, 1 / 48], rtol=2e-7)


@pytest.fixture(scope="module")
def cfg1_table():
    return build_table(unit_cell_grid(16), 64, FillSpec.random(0))


def test_cfg1_table_matches_reference(cfg1_table, golden_cfg1):
    assert sha(cfg1_table.data) == str(golden_cfg1["table_sha"])


@pytest.mark.parametrize("kind", KINDS)
def test_c_fp32_kernels_bitwise_all_512(cfg1_table, golden_cfg1, kind):
    """The C restatement of the numba fp32 kernels is bitwise equal to the
    reference on every output of config 1 (sha over [512][S][64])."""
    out = oracle.eval_f32(kind, cfg1_table.data, cfg1_table.grid.spacings, golden_cfg1["positions"])
    assert sha(out[:, :, :64]) == str(golden_cfg1[f"{kind}_f32_sha"])
    edge = oracle.eval_f32(kind, cfg1_table.data, cfg1_table.grid.spacings, golden_cfg1["edge_positions"])
    np.testing.assert_array_equal(edge[:, :, :64], golden_cfg1[f"{kind}_f32_edge"])


@pytest.mark.parametrize("kind", KINDS)
def test_c_fp32_overwrite_keeps_last(cfg1_table, golden_cfg1, kind):
    pos = golden_cfg1["positions"][:100]
    last = oracle.eval_f32(kind, cfg1_table.data, cfg1_table.grid.spacings, pos, overwrite=True, nthreads=3)
    full = oracle.eval_f32(kind, cfg1_table.data, cfg1_table.grid.spacings, pos[-1:])
    np.testing.assert_array_equal(last, full[0])


@pytest.mark.parametrize("kind", KINDS)
def test_f64_oracle_matches_reference(cfg1_table, golden_cfg1, kind):
    pos = golden_cfg1["positions"][:24]
    got, scale = oracle.eval_f64(kind, cfg1_table.data, 64, cfg1_table.grid.spacings, pos)
    np.testing.assert_array_equal(got, golden_cfg1[f"{kind}_f64_head"])
    edge, _ = oracle.eval_f64(kind, cfg1_table.data, 64, cfg1_table.grid.spacings, golden_cfg1["edge_positions"])
    np.testing.assert_array_equal(edge, golden_cfg1[f"{kind}_f64_edge"])
    assert (scale >= np.abs(got) * (1 - 1e-12)).all()
    npy = oracle.evaluate_f64_np(kind, cfg1_table.data, 64, cfg1_table.grid.spacings, pos[:4])
    np.testing.assert_array_equal(npy, got[:4])


def test_reference_fp32_within_tolerance_of_f64(cfg1_table, golden_cfg1):
    """the reference's own fp32 kernels sit well inside 1e-5 sum|w c|."""
    pos = golden_cfg1["positions"][:64]
    for kind in KINDS:
        ref, scale = oracle.eval_f64(kind, cfg1_table.data, 64, cfg1_table.grid.spacings, pos)
        ok, worst = oracle.tolerance_check(golden_cfg1[f"{kind}_f32_head"], ref, scale, 1e-5)
        assert ok and worst < 0.1, worst


@pytest.mark.parametrize("tag", ["ragged5", "g12n24", "g5x4x6n7", "g8n33"])
def test_small_cases(golden_small, tag):
    meta = golden_small[f"{tag}_meta"]
    counts, n, seed = tuple(int(x) for x in meta[:3]), int(meta[3]), int(meta[4])
    spac = tuple(float(x) for x in golden_small[f"{tag}_spacing"])
    table = build_table(GridSpec(*counts, *spac), n, FillSpec.random(seed))
    assert sha(table.data) == str(golden_small[f"{tag}_table_sha"])
    pos = golden_small[f"{tag}_positions"]
    for kind in KINDS:
        f32 = oracle.eval_f32(kind, table.data, spac, pos)
        np.testing.assert_array_equal(f32[:, :, :n], golden_small[f"{tag}_{kind}_f32"])
        f64, _ = oracle.eval_f64(kind, table.data, n, spac, pos)
        np.testing.assert_array_equal(f64, golden_small[f"{tag}_{kind}_f64"])

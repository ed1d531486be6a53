"""The product's seeded input generators reproduce the reference's inputs
(tables, position streams) -- pinned by fixtures made from the reference.
Also pins, on the CPU, the Philox4x64-10 algorithm that the device fill
kernel (csrc/spo_table.cu) implements."""
import hashlib

import numpy as np

from paper_1611_02665_b200.coeffs import FillSpec, build_table, spline_keys
from paper_1611_02665_b200.grid import GridSpec, unit_cell_grid
from paper_1611_02665_b200.workloads import CONFIGS, config_positions, generate_positions, position_stream

M64 = (1 << 64) - 1


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def philox4x64_10(ctr, key):
    """Restatement of csrc/spo_table.cu philox4x64_10 (numpy philox.h)."""
    M0, M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
    W0, W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B
    c, k0, k1 = list(ctr), key[0], key[1]
    for r in range(10):
        if r:
            k0, k1 = (k0 + W0) & M64, (k1 + W1) & M64
        p0, p1 = M0 * c[0], M1 * c[2]
        c = [(p1 >> 64) ^ c[1] ^ k0, p1 & M64, (p0 >> 64) ^ c[3] ^ k1, p0 & M64]
    return c


def device_fill_model(seed, n, count):
    """What fill_uniform_kernel computes for spline n, elements 0..count-1."""
    k = [int(x) for x in spline_keys(seed, n + 1)[n]]
    out = np.empty(count, dtype=np.float32)
    for e in range(count):
        w = philox4x64_10([(e >> 3) + 1, 0, 0, 0], k)[(e >> 1) & 3]
        u = (w >> 32) if (e & 1) else (w & 0xFFFFFFFF)
        r = np.float32(u >> 8) * np.float32(1.0 / 16777216.0)
        out[e] = r * np.float32(2.0) - np.float32(1.0)
    return out


def test_device_philox_algorithm_matches_numpy(golden_philox):
    for n in (0, 1, 63, 4095):
        ref = golden_philox[f"fill_s0_n{n}"].reshape(-1)
        idx = np.r_[0:40, ref.size - 9: ref.size]
        model = device_fill_model(0, n, ref.size if ref.size < 64 else 40)
        np.testing.assert_array_equal(model, ref[: model.size])
        # tail elements (counter > 1 block): evaluate the model directly
        k = [int(x) for x in spline_keys(0, n + 1)[n]]
        for e in idx[40:]:
            w = philox4x64_10([(int(e) >> 3) + 1, 0, 0, 0], k)[(int(e) >> 1) & 3]
            u = (w >> 32) if (e & 1) else (w & 0xFFFFFFFF)
            v = np.float32(u >> 8) * np.float32(1.0 / 16777216.0) * np.float32(2.0) - np.float32(1.0)
            assert v == ref[e]


def test_fillspec_matches_reference(golden_philox):
    g = unit_cell_grid(16)
    for n in (0, 1, 63, 4095):
        np.testing.assert_array_equal(FillSpec.random(0).spline_values(g, n), golden_philox[f"fill_s0_n{n}"])
    np.testing.assert_array_equal(FillSpec.random(7).spline_values(GridSpec(5, 4, 6), 5),
                                  golden_philox["fill_s7_n5_g5x4x6"])


def test_position_streams_match_reference(golden_philox, golden_cfg1):
    np.testing.assert_array_equal(position_stream(1, 3, 2, 2, 37, unit_cell_grid(16)),
                                  golden_philox["pos_s1_w3_i2_k2"])
    np.testing.assert_array_equal(position_stream(1, 4095, 0, 2, 256, unit_cell_grid(64)),
                                  golden_philox["pos_s1_w4095_i0_k2"])
    np.testing.assert_array_equal(generate_positions(1, 0, 0, 512, unit_cell_grid(16)).vgh,
                                  golden_cfg1["positions"])
    np.testing.assert_array_equal(config_positions(CONFIGS[1])["vgh"], golden_cfg1["positions"])


def test_config_positions_match_reference(golden_big):
    for tag, idx in (("cfg2", 2), ("cfg3", 3), ("cfg4", 4)):
        cfg = CONFIGS[idx]
        p = config_positions(cfg, walkers=[0, cfg.walkers - 1])[cfg.kernel]
        ref = golden_big[f"{tag}_positions"]
        np.testing.assert_array_equal(p[:4], ref[:4])
        np.testing.assert_array_equal(p[cfg.moves: cfg.moves + 4], ref[4:])


def test_config_shapes():
    c2 = config_positions(CONFIGS[2], walkers=range(2))
    assert c2["vgh"].shape == (2 * 64, 3) and c2["v"].shape == (2 * 32 * 12, 3)
    c5 = config_positions(CONFIGS[5], walkers=range(3))
    assert sum(v.shape[0] for v in c5.values()) == 3 * 128
    assert c5["vgl"].shape[0] == sum(1 for i in range(384) if i % 14 == 12)


def test_build_table_matches_reference_small(golden_small, golden_cfg1):
    t = build_table(unit_cell_grid(16), 64, FillSpec.random(0))
    assert sha(t.data) == str(golden_cfg1["table_sha"])

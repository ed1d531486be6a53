"""On-device input generation and the tile autotuner."""
import numpy as np
import pytest

from paper_1611_02665_b200.device import DeviceTable
from paper_1611_02665_b200.grid import GridSpec, unit_cell_grid
from paper_1611_02665_b200.tune import tile_candidates, tune_tile_size
from paper_1611_02665_b200.workloads import device_walker_positions, walker_positions

pytestmark = pytest.mark.gpu


def test_device_positions_bitwise(golden_philox):
    g64 = unit_cell_grid(64)
    got = device_walker_positions(1, 4095, 1, 0, "vgh", 256, g64).cpu().numpy()
    np.testing.assert_array_equal(got, golden_philox["pos_s1_w4095_i0_k2"])
    g16 = unit_cell_grid(16)
    got = device_walker_positions(1, 3, 1, 2, "vgh", 37, g16).cpu().numpy()
    np.testing.assert_array_equal(got, golden_philox["pos_s1_w3_i2_k2"])
    g = GridSpec(7, 9, 11, 0.3, 0.7, 1.9)
    for kind in ("v", "vgl", "vgh"):
        got = device_walker_positions(12345, 100, 64, 5, kind, 33, g).cpu().numpy()
        np.testing.assert_array_equal(got, walker_positions(12345, range(100, 164), 5, kind, 33, g))


def test_tile_autotuner():
    assert tile_candidates(256) == [32, 64, 128, 256]
    dt = DeviceTable.random(unit_cell_grid(24), 256, seed=0, tile_size=None)
    res = tune_tile_size(dt, "vgh", n_positions=8192, repeats=2)
    assert res.scanned == (32, 64, 128, 256)
    assert res.best_tile in res.scanned and len(res.throughputs) == 4
    assert res.best_throughput == max(res.throughputs)
    assert all(t > 0 for t in res.throughputs)
    # opt-in k-power form: every candidate carries it and is timed on it
    res_kp = tune_tile_size(dt, "vgh", n_positions=2 * 24 ** 3, repeats=2, kpower=True)
    assert res_kp.scanned == (32, 64, 128, 256) and all(t > 0 for t in res_kp.throughputs)

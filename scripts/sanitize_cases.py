#!/usr/bin/env python
"""Small cases for compute-sanitizer (memcheck / racecheck / initcheck):
config 1 (16^3, N=64) and ragged tables (N=5, 24, 33; non-cubic grids), every
kernel kind, fast (TMA + generic) and strict modes, tiled tables, fp64, the
table pack/fill kernels and the prologue.  Exits non-zero on a mismatch.

    compute-sanitizer --tool memcheck python scripts/sanitize_cases.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_1611_02665_b200 import DeviceTable, FillSpec, GridSpec, build_table, evaluate
    from paper_1611_02665_b200.grid import map_to_grid, unit_cell_grid

    rng = np.random.default_rng(0)
    cases = [(unit_cell_grid(16), 64), (GridSpec(12, 12, 12), 5), (GridSpec(12, 12, 12), 24),
             (GridSpec(8, 9, 10, 0.5, 0.25, 2.0), 33)]
    for grid, n in cases:
        host = build_table(grid, n, FillSpec.random(3))
        pos = rng.random((37, 3)) * np.asarray(grid.lengths) * 2.0 - 0.5
        for tile in (None, 16):
            dt = DeviceTable.from_host(host, tile_size=tile)
            for kind in ("v", "vgl", "vgh"):
                a = evaluate(dt, kind, pos, pipeline=True)
                b = evaluate(dt, kind, pos, pipeline=False)
                c = evaluate(dt, kind, pos, mode="strict")
                assert torch.equal(a, b), (grid, n, tile, kind)
                assert torch.isfinite(c).all()
        rnd = DeviceTable.random(grid, n, seed=3)
        assert torch.equal(rnd.data, DeviceTable.from_host(host).data)
        f64 = DeviceTable.normal_f64(grid, n, seed=1, tile_size=16)
        for kind in ("v", "vgl", "vgh"):
            assert torch.isfinite(evaluate(f64, kind, pos)).all()
    map_to_grid((0.3, 0.7, 0.9), unit_cell_grid(16))
    torch.cuda.synchronize()
    print("sanitize cases ok")


if __name__ == "__main__":
    main()

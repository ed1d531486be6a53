#!/usr/bin/env python
"""A few identical evaluate() launches for an ncu capture:
    python scripts/micro/one_launch.py grid N kind density [f32|f64] [bspline|kpower] [line|window|tma]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main():
    import torch

    from paper_1611_02665_b200 import DeviceTable, evaluate
    from paper_1611_02665_b200.grid import unit_cell_grid

    n_grid, n, kind, dens = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], float(sys.argv[4])
    f64 = len(sys.argv) > 5 and sys.argv[5] == "f64"
    form = sys.argv[6] if len(sys.argv) > 6 else "bspline"
    if len(sys.argv) > 7:
        os.environ["SPO_LINE"] = {"line": "1", "window": "2"}.get(sys.argv[7], "0")
    grid = unit_cell_grid(n_grid)
    dt = DeviceTable.normal_f64(grid, n, seed=1) if f64 else DeviceTable.random(grid, n, seed=1)
    if form == "kpower":
        dt.with_kpower()
    P = int(dens * n_grid ** 3)
    pos = torch.from_numpy(np.random.default_rng(P).random((P, 3))).cuda()
    S = {"v": 1, "vgl": 5, "vgh": 10}[kind]
    out = torch.empty((P, S, dt.lanes), device="cuda", dtype=dt.data.dtype)
    for _ in range(4):
        evaluate(dt, kind, pos, out, check=False, form=form, pipeline=True)
    torch.cuda.synchronize()
    print("done", P)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Fixed-cost breakdown of the TMA-pipelined path at small batches (run under
ncu --metrics gpu__time_duration.sum for the per-kernel split)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main():
    import torch

    from paper_1611_02665_b200 import DeviceTable, evaluate
    from paper_1611_02665_b200.grid import unit_cell_grid

    for n_grid, n, P in ((16, 64, 256), (48, 512, 4096)):
        dt = DeviceTable.random(unit_cell_grid(n_grid), n, seed=0)
        pos = torch.from_numpy(np.random.default_rng(P).random((P, 3))).cuda()
        out = torch.empty((P, 10, dt.lanes), device="cuda")
        for _ in range(3):
            evaluate(dt, "vgh", pos, out, pipeline=True, check=False)
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()

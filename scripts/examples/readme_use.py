"""The README's "Use" snippet, runnable (python scripts/examples/readme_use.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import paper_1611_02665_b200 as bspb

grid = bspb.unit_cell_grid(64)
table = bspb.DeviceTable.random(grid, 4096, seed=0)
pos = bspb.workloads.device_walker_positions(1, 0, 256, 0, "vgh", 256, grid)
out = bspb.evaluate_vgh(table, pos)
s = bspb.streams(out, table, "vgh")
print(tuple(out.shape), sorted(s)[:3], s["v"].shape, bspb.kernels.eval_path(table, "vgh", pos.shape[0]))

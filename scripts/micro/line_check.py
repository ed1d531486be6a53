#!/usr/bin/env python
"""Line-window kernel vs the per-position TMA kernel: bitwise equality and
interleaved timing (SPO_LINE=1 / 0)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main():
    import torch

    from paper_1611_02665_b200 import DeviceTable, evaluate
    from paper_1611_02665_b200.grid import unit_cell_grid

    cases = [(16, 512, 2000, "vgh", "f32"), (20, 512, 30000, "v", "f32"), (20, 1024, 30000, "vgl", "f32"),
             (24, 256, 30000, "vgh", "f64"), (48, 512, 16384, "vgh", "f32"), (48, 2048, 131072, "vgl", "f32"),
             (64, 4096, 262144, "vgh", "f32")]
    if len(sys.argv) > 1:
        cases = cases[: int(sys.argv[1])]
    for n_grid, n, P, kind, dtype in cases:
        grid = unit_cell_grid(n_grid)
        dt = DeviceTable.random(grid, n, seed=1) if dtype == "f32" else DeviceTable.normal_f64(grid, n, seed=1)
        pos = torch.from_numpy(np.random.default_rng(P).random((P, 3)) * 3.0 - 1.0).cuda()
        outs = {}
        for v in ("1", "0"):
            os.environ["SPO_LINE"] = v
            outs[v] = evaluate(dt, kind, pos, pipeline=True)
        torch.cuda.synchronize()
        same = bool(torch.equal(outs["1"], outs["0"]))
        del outs
        out = torch.empty((P, {"v": 1, "vgl": 5, "vgh": 10}[kind], dt.lanes), dtype=dt_torch(dt), device="cuda")
        times = {"1": [], "0": []}
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        for rnd in range(4):
            for v in ("1", "0"):
                os.environ["SPO_LINE"] = v
                evaluate(dt, kind, pos, out, pipeline=True, check=False)
                e0.record()
                for _ in range(reps):
                    evaluate(dt, kind, pos, out, pipeline=True, check=False)
                e1.record()
                e1.synchronize()
                if rnd:
                    times[v].append(e0.elapsed_time(e1) / reps)
        ms = {("line" if k == "1" else "tma"): round(float(np.median(t)), 4) for k, t in times.items()}
        rate = {k: P * n / (v * 1e-3) for k, v in ms.items()}
        print(json.dumps({"grid": n_grid, "N": n, "P": P, "kind": kind, "dtype": dtype, "bitwise": same,
                          "ms": ms, "evals_per_s": {k: float(f"{v:.4g}") for k, v in rate.items()}}), flush=True)


def dt_torch(dt):
    import torch

    return torch.float64 if dt.dtype.itemsize == 8 else torch.float32


if __name__ == "__main__":
    main()

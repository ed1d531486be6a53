#!/usr/bin/env python
"""V on the line kernel: SPO_VGROUP = 1, 2 or 4 consecutive positions per
consumer warp, and the per-position TMA kernel, in the sustained regime (all
variants in one process, interleaved), per density / dtype / table form.
    python scripts/micro/vm_sweep.py [grid] [N] [densities] [f32|f64] [bspline|kpower]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def rate(fn, secs=0.6):
    import torch

    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 0.3:
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k = 0
    e0.record()
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < secs:
        fn()
        k += 1
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / k


def main():
    import torch

    from paper_1611_02665_b200 import DeviceTable, evaluate
    from paper_1611_02665_b200.grid import unit_cell_grid

    n_grid = int(sys.argv[1]) if len(sys.argv) > 1 else 48
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    dens = [float(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0.5, 0.89, 2, 4]
    f64 = len(sys.argv) > 4 and sys.argv[4] == "f64"
    form = sys.argv[5] if len(sys.argv) > 5 else "bspline"
    dt = (DeviceTable.normal_f64(unit_cell_grid(n_grid), n, seed=1) if f64
          else DeviceTable.random(unit_cell_grid(n_grid), n, seed=1))
    if form == "kpower":
        dt.with_kpower()
    for d in dens:
        P = int(d * n_grid ** 3)
        pos = torch.from_numpy(np.random.default_rng(P).random((P, 3))).cuda()
        out = torch.empty((P, 1, dt.lanes), device="cuda", dtype=torch.float64 if f64 else torch.float32)
        res = {}
        groups = os.environ.get("VM_SWEEP", "1,2,4").split(",")
        for name, line, vm in [("tma", "0", "1")] + [(f"line{v}", "1", v) for v in groups] * 2:
            os.environ["SPO_LINE"], os.environ["SPO_VGROUP"] = line, vm
            res.setdefault(name, []).append(round(rate(lambda: evaluate(dt, "v", pos, out, check=False,
                                                                        form=form, pipeline=True)), 3))
        print(json.dumps({"grid": n_grid, "N": n, "dtype": "f64" if f64 else "f32", "form": form, "density": d,
                          "P": P, "ms": res}), flush=True)


if __name__ == "__main__":
    main()

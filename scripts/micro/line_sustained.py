#!/usr/bin/env python
"""Line-window vs per-position TMA kernel in the sustained (power-capped)
regime, across position densities (positions per grid cell): each variant
runs ~1.5 s of back-to-back launches; the rate is taken over the last 1 s,
with nvidia-smi clocks sampled meanwhile."""
import json
import os
import subprocess
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def clocks():
    try:
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                           capture_output=True, text=True, timeout=10)
        a, b = r.stdout.strip().split(",")[:2]
        return int(a), float(b)
    except Exception:
        return None, None


def main():
    import torch

    from paper_1611_02665_b200 import DeviceTable, evaluate
    from paper_1611_02665_b200.grid import unit_cell_grid

    n_grid, n = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (64, 4096)
    kind = sys.argv[3] if len(sys.argv) > 3 else "vgh"
    dens = [float(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 else [0.1, 0.25, 0.5, 1.0]
    f64 = len(sys.argv) > 5 and sys.argv[5] == "f64"
    dt = (DeviceTable.normal_f64(unit_cell_grid(n_grid), n, seed=1) if f64
          else DeviceTable.random(unit_cell_grid(n_grid), n, seed=1))
    cells = n_grid ** 3
    S = {"v": 1, "vgl": 5, "vgh": 10}[kind]
    for d in dens:
        P = int(d * cells)
        pos = torch.from_numpy(np.random.default_rng(P).random((P, 3))).cuda()
        out = torch.empty((P, S, dt.lanes), device="cuda", dtype=torch.float64 if f64 else torch.float32)
        res = {}
        for v in ("0", "1", "0", "1"):
            os.environ["SPO_LINE"] = v
            evaluate(dt, kind, pos, out, check=False)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            while time.perf_counter() - t0 < 0.5:
                evaluate(dt, kind, pos, out, check=False)
                torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            k = 0
            e0.record()
            t0 = time.perf_counter()
            clk = None
            while time.perf_counter() - t0 < 1.0:
                evaluate(dt, kind, pos, out, check=False)
                k += 1
                if clk is None and time.perf_counter() - t0 > 0.5:
                    clk = clocks()
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1) / k
            res.setdefault("line" if v == "1" else "tma", []).append((round(ms, 3), clk))
        print(json.dumps({"grid": n_grid, "N": n, "kind": kind, "dtype": "f64" if f64 else "f32", "density": d,
                          "P": P, "ms_mhz_w": res}), flush=True)


if __name__ == "__main__":
    main()

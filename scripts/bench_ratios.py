#!/usr/bin/env python
"""Throughput of the fused consumer epilogue (evaluate_ratios) vs evaluate()
on config 4 (64^3, N=4096 fp32, VGH): orbital-evals/s with the [P][10][N]
output stream (evaluate) and with the per-position ratios only (coef row of N
floats in, 10 doubles out per position).  Sustained back-to-back calls, as
scripts/bench_configs.py (timed())."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def main():
    import torch

    from bench_configs import timed

    from paper_1611_02665_b200 import DeviceTable, evaluate, evaluate_ratios
    from paper_1611_02665_b200.workloads import CONFIGS, device_walker_positions

    cfg = CONFIGS[4]
    dt = DeviceTable.random(cfg.grid, cfg.n_splines, seed=0)
    chunk = 1 << 18
    pos = device_walker_positions(1, 0, chunk // cfg.moves, 0, "vgh", cfg.moves, cfg.grid)
    coef = torch.randn((chunk, cfg.n_splines), dtype=torch.float32, device="cuda")
    out = torch.empty((chunk, 10, dt.lanes), dtype=torch.float32, device="cuda")
    res = {}
    for name, fn in (("evaluate (outputs to HBM)", lambda: evaluate(dt, "vgh", pos, out, check=False)),
                     ("evaluate_ratios (fused epilogue)", lambda: evaluate_ratios(dt, "vgh", pos, coef, check=False))):
        best = timed(fn, 3)
        res[name] = {"seconds": best, "orbital_evals_per_s": chunk * cfg.n_splines / best}
    print(json.dumps({"config": "cfg4 VGH, 262144 positions, N=4096", **res}, indent=1))


if __name__ == "__main__":
    main()

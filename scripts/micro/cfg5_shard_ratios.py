#!/usr/bin/env python
"""One rank's step of the orbital-sharded fused consumer at N = 8 on ONE GPU
(multi.evaluate_ratios_orbital_sharded at world 1: the all-reduce of the
(P, S) partials, 1.7 MB per step, is not in it): config 5's whole 12:1:1 mix
on a 512-spline fp64 slice, evaluate_ratios against evaluate per kind."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main():
    import torch

    from bench_configs import timed

    from paper_1611_02665_b200 import DeviceTable, evaluate, evaluate_ratios
    from paper_1611_02665_b200.workloads import CONFIGS, config_positions

    cfg = CONFIGS[5]
    n = cfg.n_splines // 8
    dt = DeviceTable.normal_f64(cfg.grid, n, seed=0)
    allpos = config_positions(cfg)
    res = {"config": f"cfg5 mix, one N/8 = {n}-spline fp64 slice, one GPU"}
    tot_e = tot_r = 0.0
    for kind in ("v", "vgl", "vgh"):
        pos = torch.from_numpy(allpos[kind]).cuda()
        P = pos.shape[0]
        S = {"v": 1, "vgl": 5, "vgh": 10}[kind]
        coef = torch.randn((P, n), dtype=torch.float64, device="cuda")
        out = torch.empty((P, S, dt.lanes), dtype=torch.float64, device="cuda")
        te = timed(lambda: evaluate(dt, kind, pos, out, pipeline=True, check=False), 3)
        tr = timed(lambda: evaluate_ratios(dt, kind, pos, coef, check=False), 3)
        res[kind] = {"positions": P, "evaluate_ms": round(te * 1e3, 3), "evaluate_ratios_ms": round(tr * 1e3, 3)}
        tot_e += te
        tot_r += tr
        del coef, out
        torch.cuda.empty_cache()
    res["step_ms"] = {"evaluate": round(tot_e * 1e3, 3), "evaluate_ratios": round(tot_r * 1e3, 3)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()

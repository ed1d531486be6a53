#!/usr/bin/env python
"""Sustained time of the per-position TMA kernel (SPO_LINE=0), the window
variant of the line kernel (2) and the line kernel (1) on sparse and
medium-density batches (interleaved, best of windows), B-spline form.

    python scripts/micro/window_ab.py [--reps 3]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))


def main():
    import torch

    from bench_configs import timed
    from paper_1611_02665_b200 import DeviceTable, evaluate
    from paper_1611_02665_b200.kernels import eval_path
    from paper_1611_02665_b200.workloads import CONFIGS, config_positions, device_walker_positions

    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--cases", default="all")
    args = ap.parse_args()
    cases = []
    c2 = CONFIGS[2]
    p2 = config_positions(c2)
    cases += [("cfg2-vgh", c2, "vgh", torch.from_numpy(p2["vgh"]).cuda(), "f32"),
              ("cfg2-v", c2, "v", torch.from_numpy(p2["v"]).cuda(), "f32")]
    for cfg_i, kind, walkers in ((4, "vgh", 512), (4, "vgh", 1024), (4, "vgh", 2048), (3, "vgl", 128),
                                 (3, "vgl", 256), (3, "vgl", 1024), (5, "vgh", 2048), (5, "v", 512),
                                 (5, "v", 2048)):
        cfg = CONFIGS[cfg_i]
        moves = cfg.moves
        pos = device_walker_positions(1, 0, walkers, 0, kind if cfg_i != 5 else "v", moves, cfg.grid)
        cases.append((f"cfg{cfg_i}-{kind}-{walkers}w", cfg, kind, pos, cfg.dtype))
    tables = {}
    for name, cfg, kind, pos, dtype in cases:
        if args.cases != "all" and name not in args.cases.split(","):
            continue
        key = cfg.index
        if key not in tables:
            tables.clear()
            torch.cuda.empty_cache()
            tables[key] = (DeviceTable.normal_f64(cfg.grid, 512 if cfg.index == 5 else cfg.n_splines, seed=0)
                           if dtype == "f64" else DeviceTable.random(cfg.grid, cfg.n_splines, seed=0))
        dt = tables[key]
        P = pos.shape[0]
        S = {"v": 1, "vgl": 5, "vgh": 10}[kind]
        out = torch.empty((P, S, dt.lanes), dtype=dt.data.dtype, device="cuda")
        res = {"case": name, "P": P, "per_cell": P / np.prod(cfg.grid.counts), "N": dt.n_splines}
        outs = {}
        for rep in range(2):
            for v in ("0", "2", "1"):
                os.environ["SPO_LINE"] = v
                path = eval_path(dt, kind, P, pipeline=True)
                t = timed(lambda: evaluate(dt, kind, pos, out, pipeline=True, check=False), args.reps)
                res[path] = min(res.get(path, 1e9), t * 1e3)
                if rep == 0:
                    outs[v] = out.clone() if P * S * dt.lanes < (1 << 31) else None
        os.environ.pop("SPO_LINE")
        if outs.get("0") is not None:
            res["bitwise"] = all(torch.equal(outs["0"], o) for o in outs.values() if o is not None)
        print(json.dumps(res), flush=True)
        del out, outs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

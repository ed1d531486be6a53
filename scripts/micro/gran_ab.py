#!/usr/bin/env python
"""A/B of the per-position path's two kernels (SPO_LINE=0 forces the
per-position path): eval_tma_kernel (SPO_GRAN=0, two 8 KB slab stages per
warp) vs eval_gran_kernel (SPO_GRAN=1, a ring of 2 KB row-group granules),
sustained, interleaved, bitwise compared.

    python scripts/micro/gran_ab.py [--reps 3]
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
    from paper_1611_02665_b200.workloads import CONFIGS, config_positions, device_walker_positions

    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    c2 = CONFIGS[2]
    p2 = config_positions(c2)
    cases = [("cfg2-vgh", c2, "vgh", torch.from_numpy(p2["vgh"]).cuda()),
             ("cfg2-v", c2, "v", torch.from_numpy(p2["v"]).cuda())]
    for cfg_i, kind, walkers in ((3, "vgl", 128), (3, "vgl", 256), (4, "vgh", 256), (4, "vgh", 512),
                                 (5, "vgh", 256), (5, "v", 256), (2, "vgl", 256)):
        cfg = CONFIGS[cfg_i]
        pos = device_walker_positions(1, 0, walkers, 0, kind if cfg_i != 5 else "v", cfg.moves, cfg.grid)
        cases.append((f"cfg{cfg_i}-{kind}-{walkers}w", cfg, kind, pos))
    tables = {}
    os.environ["SPO_LINE"] = "0"
    for name, cfg, kind, pos in cases:
        key = cfg.index
        if key not in tables:
            tables.clear()
            torch.cuda.empty_cache()
            tables[key] = (DeviceTable.normal_f64(cfg.grid, 512 if key == 5 else cfg.n_splines, seed=0)
                           if cfg.dtype == "f64" else DeviceTable.random(cfg.grid, cfg.n_splines, seed=0))
        dt = tables[key]
        P = pos.shape[0]
        S = {"v": 1, "vgl": 5, "vgh": 10}[kind]
        out = torch.empty((P, S, dt.lanes), dtype=dt.data.dtype, device="cuda")
        res = {"case": name, "P": P, "per_cell": P / np.prod(cfg.grid.counts), "N": dt.n_splines}
        outs = {}
        for rep in range(2):
            for v in ("0", "1"):
                os.environ["SPO_GRAN"] = v
                t = timed(lambda: evaluate(dt, kind, pos, out, pipeline=True, check=False), args.reps)
                k = "slab" if v == "0" else "gran"
                res[k] = min(res.get(k, 1e9), t * 1e3)
                if rep == 0:
                    outs[v] = out.clone()
        res["bitwise"] = torch.equal(outs["0"], outs["1"])
        res["gain"] = res["slab"] / res["gran"]
        print(json.dumps(res), flush=True)
        del out, outs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

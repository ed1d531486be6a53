#!/usr/bin/env python
"""Interleaved A/B of environment knobs the library reads per call
(SPO_PF, SPO_PFL, SPO_LINE, ...): sustained ms per launch (bench_configs.timed),
best of two rounds, outputs compared bitwise across the variants.

    python scripts/micro/env_ab.py --envs "SPO_PF=0;SPO_PF=1" [--cases cfg2-vgh,cfg4-vgh-512w] [--reps 3]

A case is cfgC-KIND (the config's own positions) or cfgC-KIND-Ww (W walkers
of the config's streams; config 5 uses its N/8 = 512 shard).
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

DEFAULT = "cfg2-vgh,cfg2-v,cfg3-vgl-128w,cfg3-vgl-1024w,cfg4-vgh-256w,cfg4-vgh-512w,cfg4-vgh-2048w,cfg5-vgh-256w"


def main():
    import torch

    from bench_configs import timed
    from paper_1611_02665_b200 import DeviceTable, evaluate
    from paper_1611_02665_b200.kernels import eval_path
    from paper_1611_02665_b200.workloads import CONFIGS, config_positions, device_walker_positions

    ap = argparse.ArgumentParser()
    ap.add_argument("--envs", required=True, help="';'-separated variants, each ','-separated K=V pairs")
    ap.add_argument("--cases", default=DEFAULT)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--form", default="auto", help="table form: auto (B-spline) or kpower (opt-in)")
    args = ap.parse_args()
    variants = [dict(kv.split("=") for kv in v.split(",") if kv) for v in args.envs.split(";")]
    keys = sorted({k for v in variants for k in v})
    tables = {}
    for name in args.cases.split(","):
        parts = name.split("-")
        cfg = CONFIGS[int(parts[0][3:])]
        kind = parts[1]
        if len(parts) > 2:
            w = int(parts[2][:-1])
            pos = device_walker_positions(1, 0, w, 0, kind if cfg.index != 5 else "v", cfg.moves, cfg.grid)
        else:
            pos = torch.from_numpy(config_positions(cfg)[kind]).cuda()
        if cfg.index not in tables:
            tables.clear()
            torch.cuda.empty_cache()
            tables[cfg.index] = (DeviceTable.normal_f64(cfg.grid, 512 if cfg.index == 5 else cfg.n_splines, seed=0)
                                 if cfg.dtype == "f64" else DeviceTable.random(cfg.grid, cfg.n_splines, seed=0))
        dt = tables[cfg.index]
        if args.form == "kpower":
            dt.with_kpower()
        P = pos.shape[0]
        S = {"v": 1, "vgl": 5, "vgh": 10}[kind]
        out = torch.empty((P, S, dt.lanes), dtype=dt.data.dtype, device="cuda")
        res = {"case": name, "P": P, "per_cell": round(P / np.prod(cfg.grid.counts), 3), "N": dt.n_splines}
        ref = None
        same = True
        for rnd in range(2):
            for vi, v in enumerate(variants):
                for k in keys:
                    os.environ.pop(k, None)
                os.environ.update(v)
                t = timed(lambda: evaluate(dt, kind, pos, out, pipeline=True, check=False, form=args.form), args.reps)
                label = ",".join(f"{k}={x}" for k, x in v.items()) or "default"
                res[label] = round(min(res.get(label, 1e9), t * 1e3), 4)
                if rnd == 0:
                    res.setdefault("paths", []).append(eval_path(dt, kind, P, pipeline=True))
                    if P * S * dt.lanes < (1 << 31):
                        if ref is None:
                            ref = out.clone()
                        else:
                            same = same and torch.equal(ref, out)
        for k in keys:
            os.environ.pop(k, None)
        res["bitwise"] = same
        print(json.dumps(res), flush=True)
        del out, ref
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

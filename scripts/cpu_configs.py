#!/usr/bin/env python
"""The reference CPU path on every BASELINE config ("Timing
the reference CPU path"): the C restatement of the reference fp32 kernels
(oracle/, bitwise equal to bspb's numba kernels) on a bounded sample of each
config's positions, all host threads and one thread.  Config 5 has no
reference fp64 production kernel: its row times the fp32 kernels at the same
shape (labelled so) and the fp64 oracle (evaluate_f64 restated in C) used
for the parity samples.

    python scripts/cpu_configs.py [--seconds 4] [--md out.md]

Test/measurement infrastructure: imports oracle/ as bench.py's CPU legs do.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import bench
    import oracle
    from paper_1611_02665_b200.workloads import CONFIGS, config_positions

    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=4.0)
    ap.add_argument("--md", default=None)
    args = ap.parse_args()
    rows = []
    for idx in (1, 2, 3, 4, 5):
        cfg = CONFIGS[idx]
        walkers = range(min(cfg.walkers, 64))
        table = bench.host_reference_table(cfg)  # fp32 U[-1,1): values do not change the speed
        for kind, pos in config_positions(cfg, walkers=walkers).items():
            if len(pos) == 0:
                continue
            # enough positions for ~seconds of work at any N (cycled through the
            # config's own positions)
            want = int(max(len(pos), 4e9 / cfg.n_splines / 64))
            pos = np.resize(pos, (want, 3))
            r = bench.cpu_baseline(table, cfg.grid, kind, pos, cfg.n_splines, args.seconds, one_thread_s=1.0)
            row = {"config": idx, "kind": kind, "N": cfg.n_splines, "dtype": "f32 kernels",
                   "all_threads": r["value"], "threads": r["cores"], "one_thread": r.get("value_1thread"),
                   "sample": r["sample"]}
            if cfg.dtype == "f64":
                row["dtype"] = "f32 kernels at the fp64 config's shape"
            rows.append(row)
            print(json.dumps(row), flush=True)
        if cfg.dtype == "f64":
            data = table.astype(np.float64)
            pos = config_positions(cfg, walkers=walkers)["vgh"][:64]
            t0 = time.perf_counter()
            oracle.eval_f64("vgh", data, cfg.n_splines, cfg.grid.spacings, pos, with_scale=False)
            dt = time.perf_counter() - t0
            row = {"config": idx, "kind": "vgh", "N": cfg.n_splines, "dtype": "f64 oracle (evaluate_f64, C)",
                   "all_threads": len(pos) * cfg.n_splines / dt, "threads": oracle.host_threads(),
                   "one_thread": None, "sample": f"{len(pos)} positions, {dt:.2f} s"}
            rows.append(row)
            print(json.dumps(row), flush=True)
        del table
    if args.md:
        with open(args.md, "w") as f:
            f.write("| cfg | kernel | N | arithmetic | all threads (orbital-evals/s) | threads | 1 thread | sample |\n")
            f.write("|---|---|---|---|---|---|---|---|\n")
            for r in rows:
                one = f"{r['one_thread']:.3e}" if r["one_thread"] else "—"
                f.write(f"| {r['config']} | {r['kind'].upper()} | {r['N']} | {r['dtype']} | "
                        f"{r['all_threads']:.3e} | {r['threads']} | {one} | {r['sample']} |\n")


if __name__ == "__main__":
    main()

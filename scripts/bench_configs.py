#!/usr/bin/env python
"""Throughput of every BASELINE config on one B200 (the BASELINE.md report
template): orbital-evals/s, algorithmic GB/s and the fraction of the measured
HBM bandwidth, per kernel kind.  Inputs are generated on the device with the
reference's streams (table: FillSpec.random(0); positions: walker streams,
seed 1).  Timing: CUDA events around each config's launches after a warm-up
pass: sustained back-to-back calls (see timed()), the regime of bench.py.

    python scripts/bench_configs.py [--configs 1,2,3,4,5] [--reps 3] [--md out.md]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, reps):
    """Sustained rate, the regime of bench.py's timed region: ~0.3 s of warm-up
    calls (clocks settle under the power controller), then `reps` x ~0.4 s of
    back-to-back calls timed with CUDA events; the mean seconds per call of the
    fastest window."""
    import time

    import torch

    fn()
    torch.cuda.synchronize()
    t0, k = time.perf_counter(), 0
    while time.perf_counter() - t0 < 0.3 or k < 2:
        fn()
        torch.cuda.synchronize()
        k += 1
    per = (time.perf_counter() - t0) / k
    n = max(2, int(0.4 / per))
    best = float("inf")
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3 / n)
    return best


def main():
    import torch

    from paper_1611_02665_b200 import DeviceTable, evaluate
    from paper_1611_02665_b200.multi import OrbitalPartition
    from paper_1611_02665_b200.workloads import CONFIGS, bytes_per_position, config_positions

    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--md", default=None)
    ap.add_argument("--forms", default="bspline,kpower", help="table forms to time (spo_b200.h SPO_TABLE_KPOWER)")
    args = ap.parse_args()
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        peak = float(json.load(f)["hbm_gbs"])
    rows = []
    chunk = 1 << 18  # launch-size quantum
    for idx in [int(c) for c in args.configs.split(",")]:
        cfg = CONFIGS[idx]
        if cfg.dtype == "f64":
            full = DeviceTable.normal_f64(cfg.grid, cfg.n_splines, seed=0)
            part = OrbitalPartition.make(cfg.n_splines, 8, quantum=16)
            shard = full.slice_orbitals(*part.local(0))
            del full
            tables = {"per-GPU shard (N/8 = 512)": shard}
            pos = config_positions(cfg)  # all 2,097,152 positions, 12:1:1
            item, q = 8, 16
        else:
            tables = {"full table": DeviceTable.random(cfg.grid, cfg.n_splines, seed=0)}
            pos = config_positions(cfg)
            item, q = 4, 32
        forms = args.forms.split(",")
        for (tname, dt), form in [(t, f) for t in tables.items() for f in forms]:
            if form == "kpower":
                dt.with_kpower()
            for kind, p in pos.items():
                if idx == 1:
                    p = p[:512]
                P = p.shape[0]
                dp = torch.from_numpy(np.ascontiguousarray(p)).cuda()
                S = {"v": 1, "vgl": 5, "vgh": 10}[kind]
                # positions per launch: as many as ~40 GB of outputs allow (the
                # batched driver's regime; config 4 VGH: 2^18, as bench.py on a
                # box without room for 2^19)
                item_b = 8 if cfg.dtype == "f64" else 4
                c = min(P, max(chunk, (40 << 30) // (S * dt.lanes * item_b) // chunk * chunk))
                out = torch.empty((c, S, dt.lanes), dtype=dt.data.dtype, device="cuda")

                def run():
                    for lo in range(0, P, c):
                        evaluate(dt, kind, dp[lo: lo + c], out[: min(c, P - lo)], check=False, form=form)

                t = timed(run, args.reps)
                bpp = bytes_per_position(kind, dt.n_splines, item, q)
                gbs = bpp * P / t / 1e9
                rows.append({"config": idx, "table": tname, "form": form, "kind": kind, "positions": P,
                             "n_splines": dt.n_splines, "dtype": cfg.dtype, "seconds": t,
                             "orbital_evals_per_s": P * dt.n_splines / t, "algorithmic_gbs": gbs,
                             "fraction_of_hbm": gbs / peak})
                print(json.dumps(rows[-1]), flush=True)
        del tables
        torch.cuda.empty_cache()
    if args.md:
        with open(args.md, "w") as f:
            f.write("| cfg | table | form | kernel | positions | N | dtype | time (ms) | orbital-evals/s | "
                    "algorithmic GB/s | fraction of %.1f GB/s |\n" % peak)
            f.write("|---|---|---|---|---|---|---|---|---|---|---|\n")
            for r in rows:
                f.write(f"| {r['config']} | {r['table']} | {r['form']} | {r['kind'].upper()} | {r['positions']:,} | "
                        f"{r['n_splines']} | {r['dtype']} | {r['seconds'] * 1e3:.3f} | "
                        f"{r['orbital_evals_per_s']:.3e} | {r['algorithmic_gbs']:,.0f} | "
                        f"{r['fraction_of_hbm']:.3f} |\n")


if __name__ == "__main__":
    main()

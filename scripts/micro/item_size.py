#!/usr/bin/env python
"""Sweep of the TMA kernel's item size (SPO_BP) at mid-size batches against
the automatic choice (spo_eval_tma.cu, ITEMS_PER_WARP_FULL)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main():
    import torch

    from paper_1611_02665_b200 import DeviceTable, evaluate
    from paper_1611_02665_b200.grid import unit_cell_grid

    for n_grid, n, P in ((16, 64, 4096), (16, 64, 16384), (48, 512, 1024), (48, 512, 4096),
                         (48, 512, 16384), (64, 4096, 256), (64, 4096, 1024), (64, 4096, 4096),
                         (64, 4096, 16384), (64, 4096, 32768), (64, 4096, 65536)):
        dt = DeviceTable.random(unit_cell_grid(n_grid), n, seed=0)
        pos = torch.from_numpy(np.random.default_rng(P).random((P, 3))).cuda()
        out = torch.empty((P, 10, dt.lanes), device="cuda")
        variants = ("auto", 1, 2, 4, 8)
        times = {str(v): [] for v in variants}
        ref = None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(2, int(2e4 // max(P * n // 4096, 1)))
        for rnd in range(6):  # interleaved rounds: clock drift hits every variant alike
            for bp in variants:
                if bp == "auto":
                    os.environ.pop("SPO_BP", None)
                else:
                    os.environ["SPO_BP"] = str(bp)
                evaluate(dt, "vgh", pos, out, pipeline=True, check=False)
                torch.cuda.synchronize()
                if ref is None:
                    ref = out.clone()
                elif rnd == 0:
                    assert torch.equal(out, ref), bp
                e0.record()
                for _ in range(reps):
                    evaluate(dt, "vgh", pos, out, pipeline=True, check=False)
                e1.record()
                e1.synchronize()
                if rnd:
                    times[str(bp)].append(e0.elapsed_time(e1) / reps * 1e3)
        res = {k: round(float(np.median(v)), 1) for k, v in times.items()}
        os.environ.pop("SPO_BP", None)
        print(json.dumps({"grid": n_grid, "N": n, "P": P, "us_per_call": res}), flush=True)


if __name__ == "__main__":
    main()

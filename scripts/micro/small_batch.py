#!/usr/bin/env python
"""Per-call latency of evaluate() vs batch size, TMA-pipelined vs generic
kernel, eager and CUDA-graph replayed (decides the small-batch cutover in
kernels.evaluate)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main():
    import torch

    from paper_1611_02665_b200 import DeviceTable, evaluate
    from paper_1611_02665_b200.graphs import GraphedEvaluator
    from paper_1611_02665_b200.grid import unit_cell_grid

    for n_grid, n in ((16, 64), (48, 512), (64, 4096)):
        dt = DeviceTable.random(unit_cell_grid(n_grid), n, seed=0)
        for P in (1, 8, 64, 256, 1024, 4096, 16384):
            pos = torch.from_numpy(np.random.default_rng(P).random((P, 3))).cuda()
            out = torch.empty((P, 10, dt.lanes), device="cuda")
            res = {}
            for pipe in (True, False):
                for _ in range(3):
                    evaluate(dt, "vgh", pos, out, pipeline=pipe, check=False)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                reps = 20
                e0.record()
                for _ in range(reps):
                    evaluate(dt, "vgh", pos, out, pipeline=pipe, check=False)
                e1.record()
                e1.synchronize()
                res["tma" if pipe else "generic"] = e0.elapsed_time(e1) / reps * 1e3
                g = GraphedEvaluator(dt, "vgh", P, pipeline=pipe)
                for _ in range(3):
                    g.run(pos)
                torch.cuda.synchronize()
                e0.record()
                for _ in range(reps):
                    g.run(pos)
                e1.record()
                e1.synchronize()
                res[("tma" if pipe else "generic") + "_graph"] = e0.elapsed_time(e1) / reps * 1e3
            print(json.dumps({"grid": n_grid, "N": n, "P": P, "us_per_call": res}), flush=True)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Sustained time per call of small batches three ways: evaluate() back to
back, the same captured in a CUDA graph (GraphedEvaluator, one graph launch
per call), and one graph holding 20 calls (launch gaps between the calls'
kernels only).  Shows how much of a small batch's time is host / launch
overhead rather than kernel time.

    python scripts/micro/launch_overhead.py
"""
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
    from paper_1611_02665_b200.graphs import GraphedEvaluator
    from paper_1611_02665_b200.kernels import eval_path
    from paper_1611_02665_b200.workloads import CONFIGS, config_positions

    for cfg_i, kind in ((2, "vgh"), (2, "v"), (3, "vgl")):
        cfg = CONFIGS[cfg_i]
        dt = DeviceTable.random(cfg.grid, cfg.n_splines, seed=0)
        pos = torch.from_numpy(config_positions(cfg)[kind]).cuda()
        if cfg_i == 3:
            pos = pos[:16384].contiguous()
        P = pos.shape[0]
        S = {"v": 1, "vgl": 5, "vgh": 10}[kind]
        out = torch.empty((P, S, dt.lanes), dtype=torch.float32, device="cuda")
        t_eval = timed(lambda: evaluate(dt, kind, pos, out, check=False), 3)
        ge = GraphedEvaluator(dt, kind, P)
        ge.positions.copy_(pos)
        t_graph = timed(lambda: ge.graph.replay(), 3)
        g20 = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            evaluate(dt, kind, pos, out, check=False)
        torch.cuda.current_stream().wait_stream(side)
        with torch.cuda.graph(g20):
            for _ in range(20):
                evaluate(dt, kind, pos, out, check=False)
        t_g20 = timed(lambda: g20.replay(), 3) / 20
        print(json.dumps({"case": f"cfg{cfg_i}-{kind}", "P": P, "path": eval_path(dt, kind, P),
                          "evaluate_ms": t_eval * 1e3, "graph_ms": t_graph * 1e3, "graph20_ms_per_call": t_g20 * 1e3}),
              flush=True)
        del dt, out, ge, g20
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

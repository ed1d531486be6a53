"""Where the drop-in call's time goes: eval_batch on the bench workload
(config 4, host positions, k-power table), per-call wall times and a
cProfile of one call."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main():
    import torch

    from paper_1611_02665_b200 import DeviceTable, WalkerOutputsSoA, eval_batch
    from paper_1611_02665_b200.workloads import CONFIGS, walker_positions

    cfg = CONFIGS[4]
    pos = walker_positions(1, range(0, 4096), 0, "vgh", cfg.moves, cfg.grid)
    dt = DeviceTable.random(cfg.grid, cfg.n_splines, seed=0)
    if len(sys.argv) > 1 and sys.argv[1] == "kpower":
        dt.with_kpower()
    out = WalkerOutputsSoA(cfg.n_splines)
    eval_batch(dt, "vgh", pos, out)
    torch.cuda.synchronize()
    for _ in range(3):
        t0 = time.perf_counter()
        eval_batch(dt, "vgh", pos, out)
        print("eval_batch", (time.perf_counter() - t0) * 1e3, "ms", flush=True)
    pr = cProfile.Profile()
    pr.enable()
    eval_batch(dt, "vgh", pos, out)
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(18)


if __name__ == "__main__":
    main()

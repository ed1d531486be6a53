#!/usr/bin/env python
"""Randomised stress of the line-window kernel's synchronisation (plane ring,
shared position counter, position groups): random grids, orbital counts,
kinds, dtypes, table forms and densities, each evaluated by the line kernel
(SPO_LINE=1), its window variant (SPO_LINE=2; k-power tables fall back to the
per-position kernel) and the per-position TMA kernel (SPO_LINE=0) -- the
results must be bitwise equal.  Exits non-zero on the first mismatch.

    python scripts/stress_line.py [iterations] [seed]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_1611_02665_b200 import DeviceTable, evaluate
    from paper_1611_02665_b200.grid import GridSpec

    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    t0 = time.time()
    for it in range(iters):
        n3 = [int(x) for x in rng.integers(4, 41, size=3)]
        f64 = bool(rng.random() < 0.3)
        q = 16 if f64 else 32
        n = int(rng.integers(1, 9)) * (64 if f64 else 128) - int(rng.integers(0, q))
        grid = GridSpec(*n3, 1.0 / n3[0], 1.0 / n3[1], 1.0 / n3[2])
        tile = [None, "auto"][int(rng.integers(0, 2))]
        dt = (DeviceTable.normal_f64(grid, n, seed=it, tile_size=tile) if f64
              else DeviceTable.random(grid, n, seed=it, tile_size=tile))
        form = "kpower" if rng.random() < 0.5 else "bspline"
        if form == "kpower":
            dt.with_kpower()
        kind = ["v", "vgl", "vgh"][int(rng.integers(0, 3))]
        dens = float(rng.choice([0.05, 0.15, 0.3, 0.8, 1.5, 3.0, 6.0, 17.0]))
        P = max(1, int(dens * np.prod(n3))) + int(rng.integers(0, 64))
        # three full outputs are alive at once: keep each under 8 GB
        S = {"v": 1, "vgl": 5, "vgh": 10}[kind]
        P = min(P, int(8e9 / (S * (n + q) * (8 if f64 else 4))))
        pos = rng.random((P, 3)) * 3.0 - 1.0
        if rng.random() < 0.2:
            pos[rng.integers(0, P, size=3), rng.integers(0, 3, size=3)] = np.nan
        dpos = torch.from_numpy(pos).cuda()
        outs = []
        for line in ("1", "2", "0"):
            os.environ["SPO_LINE"] = line
            st = torch.zeros(1, dtype=torch.int32, device="cuda")
            outs.append(evaluate(dt, kind, dpos, pipeline=True, form=form, status=st, check=False))
        torch.cuda.synchronize()
        b = outs[2].nan_to_num(123.0)
        ok = all(bool(torch.equal(o.nan_to_num(123.0), b)) for o in outs[:2])
        print(f"{it:3d} grid={n3} N={n} {'f64' if f64 else 'f32'} tile={tile} {form} {kind} P={P} "
              f"({dens}/cell) {'ok' if ok else 'MISMATCH'}", flush=True)
        if not ok:
            return 1
        del dt, outs, b
        torch.cuda.empty_cache()
    print(f"all {iters} cases bitwise equal ({time.time() - t0:.0f} s)")
    return 0


if __name__ == "__main__":
    sys.exit(main())

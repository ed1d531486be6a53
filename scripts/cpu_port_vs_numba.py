#!/usr/bin/env python
"""The reference arm's fidelity: the C restatement of the reference fp32
kernels (oracle/spline_oracle.c, what bench.py --impl reference and
cpu_baseline time on the GPU box) against the reference's own numba kernels
(bspb.kernels.eval_batch), same table, positions and thread counts.  Needs
/root/reference (this container only; the GPU box has no numba build of the
reference).  One batch per thread, reference batch semantics (each worker
overwrites its output), orbital-evals/s = positions * N / wall.

    python scripts/cpu_port_vs_numba.py [grid N kind ...]
"""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")


def main():
    from bspb.coeffs import FillSpec, build_table
    from bspb.grid import GridSpec
    from bspb.kernels import KernelKind, allocate_outputs, eval_batch

    import oracle

    cases = [(64, 4096, "vgh", 600), (48, 2048, "vgl", 1500), (48, 512, "v", 20000)]
    threads = len(os.sched_getaffinity(0))
    print(f"host threads: {threads}")
    for n, N, kind, per_thread in cases:
        grid = GridSpec(n, n, n, 1 / n, 1 / n, 1 / n)
        table = build_table(grid, N, FillSpec.linear_index("x"))  # values do not change the speed
        data = np.asarray(table.data)
        k = KernelKind(kind)
        for nt in (1, threads):
            pos = [np.random.default_rng(t).random((per_thread, 3)) for t in range(nt)]
            outs = [allocate_outputs(table) for _ in range(nt)]
            eval_batch(table, k, pos[0][:8], outs[0])  # JIT warm
            with ThreadPoolExecutor(nt) as ex:
                t0 = time.perf_counter()
                list(ex.map(lambda a: eval_batch(table, k, a[0], a[1]), zip(pos, outs)))
                numba = nt * per_thread * N / (time.perf_counter() - t0)
            allp = np.concatenate(pos)
            oracle.eval_f32(kind, data, grid.spacings, allp[:8], overwrite=True, nthreads=nt)
            t0 = time.perf_counter()
            oracle.eval_f32(kind, data, grid.spacings, allp, overwrite=True, nthreads=nt)
            port = nt * per_thread * N / (time.perf_counter() - t0)
            print(f"{n}^3 N={N} {kind.upper():3s} threads={nt:2d}  numba {numba:.3e}  C port {port:.3e}  "
                  f"port/numba {port / numba:.2f}", flush=True)


if __name__ == "__main__":
    main()

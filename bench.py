#!/usr/bin/env python
"""Benchmark: B-spline VGH orbital-evals/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config 4] [--chunk 0] [--mode fast] [--tile 0]

Workload (default, BASELINE config 4 -- the VGH config with N >= 2048 the
north-star roofline target names): 64^3 periodic grid (67^3 wrap-padded),
N = 4096 fp32 orbitals, FillSpec.random(0) table (generated on the device,
bit-identical to the reference's numpy fill), 4096 walkers x 256 moves =
1,048,576 VGH positions per GPU per step (Philox walker streams, seed 1).
A step evaluates all of them, in launches of `--chunk` positions into a
reusable output buffer (every output is written to HBM; the reference also
overwrites its output buffer per position, kernels.py:353-354).  --chunk 0
(default): 524,288 positions per launch (2 per grid cell: more stencil planes
shared by the line kernel) when the GPU has room for the 86 GB output buffer,
else 262,144.

Multi-GPU (torchrun, one rank per GPU): walker-sharded, table replicated,
each rank evaluates its own 4096-walker population (weak scaling), no
collective on the data path; time = max over ranks.

Printed JSON (rank 0): value = orbital-evals/s over all ranks; roofline of
the eval kernel (algorithmic bytes 64*Npad*4 + 10*Npad*4 per position over
the measured HBM copy bandwidth); e2e through the drop-in API eval_batch with
host buffers; cpu_baseline = the C restatement of the reference fp32 kernels
(oracle/, kind "port") on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "B-spline VGH orbital-evals/s"
UNIT = "orbital-evals/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--kind", default=None, help="override the config kernel (v/vgl/vgh)")
    ap.add_argument("--chunk", type=int, default=0, help="positions per launch (0 = auto)")
    ap.add_argument("--mode", default="fast", choices=("fast", "strict"))
    ap.add_argument("--tile", type=int, default=-1, help="AoSoA tile size (-1 = auto, 0 = untiled)")
    ap.add_argument("--form", default="auto", choices=("auto", "kpower", "bspline"),
                    help="device table form of FAST evaluations (spo_b200.h SPO_TABLE_KPOWER); auto = "
                         "k-power form for dense (line-kernel) batches")
    ap.add_argument("--walkers", type=int, default=0, help="override walkers per GPU")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline sample budget")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t0=None, t1=None):
        """Median SM clock and active throttle reasons over samples taken in
        [t0, t1] (the timed region), falling back to all samples under load."""
        sm, pw, mx, reasons = [], [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        lines = [ln for ts, ln in self.lines if t0 is None or t0 - 0.25 <= ts <= t1 + 0.25]
        window = "timed region"
        if len(lines) < 2:
            lines = [ln for _, ln in self.lines]
            window = "warm-up + timed region"
        for ln in lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                pw.append(float(f[3]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for name, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "power_w": statistics.median(pw), "samples": len(sm), "window": window}


def workload(args, rank):
    from paper_1611_02665_b200.workloads import CONFIGS, bytes_per_position, walker_positions

    cfg = CONFIGS[args.config]
    if cfg.dtype != "f32" or cfg.index == 5:
        raise SystemExit("bench.py times the fp32 walker-sharded configs (1-4)")
    kind = args.kind or ("vgh" if cfg.kernel == "vgh" else cfg.kernel)
    walkers = args.walkers or cfg.walkers
    first = rank * walkers
    pos = walker_positions(1, range(first, first + walkers), 0, kind, cfg.moves, cfg.grid)
    return cfg, kind, pos, bytes_per_position(kind, cfg.n_splines)


def cpu_baseline(table_soa, grid, kind, pos, n_splines, budget_s, threads=0, one_thread_s=0.0):
    """Reference fp32 kernels restated in C (oracle/), all host threads, with
    the reference's batch semantics (each thread overwrites its own output
    buffer, kernels.py:353-354).  Calibrated to ~budget_s of CPU work."""
    import oracle

    threads = threads or oracle.host_threads()
    spac = grid.spacings
    oracle.eval_f32(kind, table_soa, spac, pos[: 4 * threads], overwrite=True, nthreads=threads)  # warm
    n = 8 * threads
    while True:
        t0 = time.perf_counter()
        oracle.eval_f32(kind, table_soa, spac, pos[:n], overwrite=True, nthreads=threads)
        dt = time.perf_counter() - t0
        if dt > 0.5 or n >= pos.shape[0]:
            break
        n = min(pos.shape[0], n * 4)
    n_final = int(min(pos.shape[0], max(n, n * budget_s / max(dt, 1e-6))))
    t0 = time.perf_counter()
    oracle.eval_f32(kind, table_soa, spac, pos[:n_final], overwrite=True, nthreads=threads)
    dt = time.perf_counter() - t0
    res = {"value": n_final * n_splines / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{n_final} of the workload's positions x N={n_splines} {kind.upper()}, "
                      f"{dt:.1f} s, C restatement of kernels.py fp32 kernels (oracle/spline_oracle.c, "
                      f"-O3 AVX2/AVX-512 clones, OpenMP)"}
    if threads > 1 and one_thread_s > 0:  # report 1-thread and all-core figures
        n1 = max(1, int(n_final / threads * one_thread_s / max(dt, 1e-6)))
        t0 = time.perf_counter()
        oracle.eval_f32(kind, table_soa, spac, pos[:n1], overwrite=True, nthreads=1)
        res["value_1thread"] = n1 * n_splines / (time.perf_counter() - t0)
    return res


def host_reference_table(cfg, seed=0):
    """Reference-layout fp32 table with U[-1,1) values for the CPU arms
    (values do not change the reference kernels' speed)."""
    from paper_1611_02665_b200.coeffs import padded_count

    nx, ny, nz = cfg.grid.counts
    npad = padded_count(cfg.n_splines)
    rng = np.random.default_rng(seed)
    data = rng.random((nx, ny, nz, npad), dtype=np.float32)
    data *= np.float32(2.0)
    data -= np.float32(1.0)
    data[..., cfg.n_splines:] = 0.0
    return data


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    from paper_1611_02665_b200.workloads import CONFIGS, walker_positions

    import oracle

    cfg = CONFIGS[args.config]
    kind = args.kind or cfg.kernel
    threads = oracle.host_threads()
    table = host_reference_table(cfg)
    # each step: a bounded sample of the workload, sized to ~ budget seconds
    per_step_budget = max(1.0, min(8.0, 150.0 / max(1, args.steps + args.warmup)))
    pos = walker_positions(1, range(0, 256), 0, kind, cfg.moves, cfg.grid)
    probe = cpu_baseline(table, cfg.grid, kind, pos, cfg.n_splines, 1.0, threads)
    n = int(min(pos.shape[0], max(threads, probe["value"] / cfg.n_splines * per_step_budget)))
    sample = pos[:n]
    for _ in range(args.warmup):
        oracle.eval_f32(kind, table, cfg.grid.spacings, sample, overwrite=True, nthreads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.eval_f32(kind, table, cfg.grid.spacings, sample, overwrite=True, nthreads=threads)
    dt = time.perf_counter() - t0
    value = n * cfg.n_splines * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC if kind == "vgh" else f"B-spline {kind.upper()} orbital-evals/s",
        "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (U[-1,1) table, Philox walker positions)",
        "config": {"workload": f"cfg{cfg.index}: {cfg.description}", "positions_per_step": n,
                   "grid": list(cfg.grid.counts), "n_splines": cfg.n_splines, "kernel": kind},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{n} positions per step x {args.steps} steps; reference fp32 kernels "
                                   "restated in C (oracle/spline_oracle.c), reference has no C build "
                                   "(numba JIT, cannot travel)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_b200(args):
    import torch

    world, rank, local = dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py --impl b200 needs a CUDA device")
    n_dev = torch.cuda.device_count()
    shared = world > n_dev  # more ranks than GPUs: a functional run only, never a measurement
    if shared:
        print(f"bench.py: {world} ranks on {n_dev} GPU(s): ranks share devices (gloo plumbing), "
              "not a scaling measurement", file=sys.stderr, flush=True)
        local %= n_dev
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        # one rank per GPU over NCCL; NCCL refuses two ranks on one device
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    from paper_1611_02665_b200 import DeviceTable, KernelKind, WalkerOutputsSoA, eval_batch, evaluate

    cfg, kind, pos_np, bpp = workload(args, rank)
    P = pos_np.shape[0]
    N = cfg.n_splines
    S = KernelKind(kind).output_streams_soa
    tile = "auto" if args.tile < 0 else (args.tile or None)
    table = DeviceTable.random(cfg.grid, N, seed=0, tile_size=tile, device=dev)
    form = args.form if args.mode == "fast" else "bspline"
    if form != "bspline":
        table.with_kpower()
    pos = torch.from_numpy(pos_np).to(dev)
    chunk = args.chunk
    if chunk <= 0:  # largest of 2^19 / 2^18 whose output buffer leaves 40 GB free
        free, _ = torch.cuda.mem_get_info(dev)
        per_pos = S * table.lanes * 4
        chunk = 1 << 19 if free - (1 << 19) * per_pos > (40 << 30) else 1 << 18
    chunk = min(chunk, P)
    out = torch.empty((chunk, S, table.lanes), dtype=torch.float32, device=dev)
    bounds = [(lo, min(P, lo + chunk)) for lo in range(0, P, chunk)]
    stream = torch.cuda.current_stream(dev)

    def step(events=None):
        for b, (lo, hi) in enumerate(bounds):
            if events is not None:
                events[b][0].record(stream)
            evaluate(table, kind, pos[lo:hi], out, mode=args.mode, check=False, form=form)
            if events is not None:
                events[b][1].record(stream)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize(dev)

    # correctness guard on the benchmarked configuration (one launch)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    evaluate(table, kind, pos[:chunk], out, mode=args.mode, status=status, check=False, form=form)
    assert int(status.item()) == 0

    launch_events = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                      for _ in bounds] for _ in range(args.steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        for _ in range(args.warmup):
            step()
        barrier()
        wall0 = time.time()
        t_start.record(stream)
        for k in range(args.steps):
            step(launch_events[k])
        t_end.record(stream)
        barrier()
        wall1 = time.time()
    elapsed_ms = t_start.elapsed_time(t_end)
    launch_ms = [s.elapsed_time(e) for ev in launch_events for (s, e) in ev]
    full = [ms for (lo, hi), ms in zip(bounds * args.steps, launch_ms) if hi - lo == chunk]
    avg_launch_ms = sum(full) / len(full)

    # max over ranks
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device="cpu" if shared else dev)
    if world > 1:
        import torch.distributed as dist

        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms = float(t.item())
    total_units = P * N * args.steps * world
    value = total_units / (elapsed_ms / 1e3)

    from paper_1611_02665_b200.kernels import eval_form, eval_path

    path = eval_path(table, kind, chunk, mode=args.mode, form=form)
    form = eval_form(table, kind, chunk, mode=args.mode, form=form)  # the form the timed launches read
    # this repo's kernels per evaluate() call (library kernels -- cub's radix
    # sort in the line path's prologue, memsets -- not counted)
    kp = "true" if form == "kpower" else "false"
    kernels_per_call, kernel_name = {
        "line": (4, f"spo::line::line_kernel<{kind.upper()},float,RATIO=false,KP={kp}> (+ line_keys, cub sort, "
                    f"line_records, line_runs prologue, timed together)"),
        "tma": (3, f"spo::tma::eval_tma_kernel<{kind.upper()},KP={kp}> (+ bucket_count, prologue_records, "
                   f"timed together)"),
        "generic": (1, f"spo::eval_kernel<{kind.upper()},float,{args.mode},KP={kp}>"),
    }[path]
    peak, peak_src = measured_peak()
    achieved = bpp * chunk / (avg_launch_ms * 1e-3) / 1e9  # GB/s per launch
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": ncu_traffic(args, cfg, kind, chunk, path, form),
                "peak_source": peak_src, "kernel": kernel_name,
                "algorithmic_bytes_per_position": bpp, "positions_per_launch": chunk,
                "avg_launch_ms": avg_launch_ms}
    if roofline["traffic"]:
        # what DRAM actually carried (ncu bytes of the same launch shape over this
        # run's launch time): frac > 1 above means the table came from L2
        roofline["dram_gbs"] = roofline["traffic"] / (avg_launch_ms * 1e-3) / 1e9
        roofline["dram_frac"] = roofline["dram_gbs"] / peak

    result = {
        "metric": METRIC if kind == "vgh" else f"B-spline {kind.upper()} orbital-evals/s",
        "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: FillSpec.random(0) table generated on device (bit-identical to the "
                "reference numpy fill), reference Philox walker position streams (seed 1)",
        "config": {"workload": f"cfg{cfg.index}: {cfg.description}", "grid": list(cfg.grid.counts),
                   "n_splines": N, "kernel": kind, "positions_per_gpu": P, "walkers_per_gpu": P // cfg.moves,
                   "chunk": chunk, "mode": args.mode, "path": path, "tile_size": table.tile_size,
                   "table_gb": table.nbytes / 1e9, "table_form": form,
                   "kpower_table_gb": (table.kdata.numel() * 4 / 1e9) if table.has_kpower else None,
                   "l2": f"inputs larger than L2 (table {table.nbytes / 1e9:.2f} GB >> 126 MB); no flush",
                   "parallelism": f"walker-sharded x{world}, table replicated"},
        "roofline": roofline,
        "gpu_launches": len(bounds) * args.steps * kernels_per_call,
        "clocks": clocks.summary(wall0, wall1),
    }

    if not args.no_e2e:
        del out  # the drop-in path sizes its own scratch from the free memory
        torch.cuda.empty_cache()
        # every rank drives its own GPU through the drop-in API at once; the
        # job's e2e time is the slowest rank's
        e2e = e2e_dropin(table, kind, pos_np, N, S, eval_batch, WalkerOutputsSoA, args, dev, world, shared)
        if rank == 0:
            result["e2e"] = e2e
            result["e2e_full_outputs"] = e2e_full_outputs(table, kind, pos_np, N, S, dev)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    if rank == 0 and world == 1 and not args.no_cpu:
        soa = table.reference_soa()
        result["cpu_baseline"] = cpu_baseline(soa, cfg.grid, kind, pos_np, N, args.cpu_seconds, one_thread_s=3.0)
        del soa
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()
    return 0


def e2e_full_outputs(table, kind, pos_np, N, S, dev, chunk=8192, seconds=2.0):
    """Transparency figure: the same metric when EVERY output is copied back to
    pinned host memory (H2D positions + kernel + D2H of all [P][S][N] outputs,
    double-buffered over two streams).  PCIe-bound by construction; measured on
    a bounded sample of the workload's positions."""
    import torch

    from paper_1611_02665_b200 import evaluate

    pin_pos = torch.from_numpy(pos_np).pin_memory()
    host = [torch.empty((chunk, S, table.lanes), dtype=torch.float32).pin_memory() for _ in range(2)]
    dout = [torch.empty((chunk, S, table.lanes), dtype=torch.float32, device=dev) for _ in range(2)]
    dpos = [torch.empty((chunk, 3), dtype=torch.float64, device=dev) for _ in range(2)]
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    n_chunks = max(2, min(len(pos_np) // chunk, 64))
    done = [torch.cuda.Event() for _ in range(2)]

    def run(k):
        b = k & 1
        with torch.cuda.stream(streams[b]):
            done[b].synchronize()
            dpos[b].copy_(pin_pos[k * chunk:(k + 1) * chunk], non_blocking=True)
            evaluate(table, kind, dpos[b], dout[b], check=False)
            host[b].copy_(dout[b], non_blocking=True)
            done[b].record(streams[b])

    run(0)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    k = 0
    while k < n_chunks and (time.perf_counter() - t0 < seconds or k < 2):
        run(k)
        k += 1
    torch.cuda.synchronize(dev)
    dt = time.perf_counter() - t0
    return {"value": k * chunk * N / dt, "unit": UNIT, "h2d_bytes_per_step": int(k * chunk * 24),
            "d2h_bytes_per_step": int(k * chunk * S * table.lanes * 4),
            "sample": f"{k} chunks of {chunk} positions, all outputs to pinned host memory"}


def e2e_dropin(table, kind, pos_np, N, S, eval_batch, WalkerOutputsSoA, args, dev, world=1, shared=False):
    """Same metric through the reference-facing drop-in call eval_batch with
    HOST buffers: host positions -> device each step, all positions evaluated,
    the last position's streams copied back into the host WalkerOutputsSoA
    (the reference API's output, kernels.py:353-354).  Timed by wall clock
    around fully synchronous calls (the call returns host data); under
    torchrun every rank runs at once and the job time is the max over ranks
    (whole-job value = all ranks' positions / that time)."""
    import torch

    out = WalkerOutputsSoA(N)
    steps = max(3, min(args.steps, 5))
    eval_batch(table, kind, pos_np, out, mode=args.mode)  # warm
    torch.cuda.synchronize(dev)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        eval_batch(table, kind, pos_np, out, mode=args.mode)
    dt = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([dt], dtype=torch.float64, device="cpu" if shared else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    P = pos_np.shape[0]
    return {"value": world * P * N * steps / dt, "unit": UNIT, "h2d_bytes_per_step": int(world * pos_np.nbytes),
            "d2h_bytes_per_step": int(world * S * table.lanes * 4), "ranks": world,
            "api": "paper_1611_02665_b200.eval_batch(table, kind, host positions, host WalkerOutputsSoA)"}


def ncu_traffic(args, cfg, kind, chunk, path, form="bspline"):
    """dram read+write bytes per launch from the committed ncu capture, when
    it was taken on this exact configuration (profiles/ncu_traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            rec = json.load(f)
        key = f"cfg{cfg.index}-{kind}-{args.mode}-tile{args.tile}-{path}-{chunk}"
        if form == "kpower":
            key += "-kpower"
        r = rec.get(key)
        if r and r.get("positions_per_launch") == chunk:
            return r["dram_bytes_per_launch"]
    except Exception:
        pass
    return None


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())

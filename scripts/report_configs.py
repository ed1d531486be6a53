#!/usr/bin/env python
"""BASELINE.md section 4 report: every config on one B200, per kernel kind,
on the default B-spline table form.

    python scripts/report_configs.py --phase time [--configs 1,2,3,4,5]   # GPU: rates + parity errors
    ncu --set full --clock-control none -k regex:"line_kernel|eval_tma_kernel|eval_kernel" \\
        -o gpurun_out/report_ncu python scripts/report_configs.py --phase ncu   # GPU: one launch each
    python scripts/report_configs.py --phase md --cpu <cpu_configs json lines>   # here: the table

time: sustained orbital-evals/s (bench_configs.timed: back-to-back launches
  after warm-up, CUDA events), algorithmic GB/s and its fraction of the
  measured HBM bandwidth, the irreducible-bytes fraction (outputs + one
  table pass), and max |got - oracle| / (tol * sum|w*c|) over a stratified
  sample of >= 2048 positions (tests/strata.py) -> gpurun_out/report_time.jsonl
ncu: the first launch of each (config, kind) in the same order and shape,
  for DRAM GB/s, L2 hit rate, FMA-pipe and L1/shared utilisation.
Config 5 is timed with the full N = 4096 fp64 table on one GPU (the
orbital-sharded run divides N across ranks; bench.py --config 5).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
OUT = os.path.join(ROOT, "gpurun_out")


def cases(configs):
    """(config, kind, table factory, positions) in report order."""
    from paper_1611_02665_b200.workloads import CONFIGS, config_positions

    for idx in configs:
        cfg = CONFIGS[idx]
        pos = config_positions(cfg)
        for kind, p in pos.items():
            if idx == 1:
                p = p[:512]
            yield cfg, kind, p


def table_for(cfg):
    from paper_1611_02665_b200 import DeviceTable

    if cfg.dtype == "f64":
        return DeviceTable.normal_f64(cfg.grid, cfg.n_splines, seed=0)
    return DeviceTable.random(cfg.grid, cfg.n_splines, seed=0)


def launch_size(P, S, lanes, item):
    """Positions per launch: as many as ~40 GB of outputs allow."""
    return int(min(P, max(1 << 18, (40 << 30) // (S * lanes * item))))


def phase_time(args):
    import torch

    import oracle
    from bench_configs import timed
    from paper_1611_02665_b200 import evaluate
    from paper_1611_02665_b200.kernels import eval_path
    from paper_1611_02665_b200.workloads import bytes_per_position
    from strata import stratified_sample

    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        peak = float(json.load(f)["hbm_gbs"])
    os.makedirs(OUT, exist_ok=True)
    rows = []
    cur, dt, host = None, None, None
    for cfg, kind, p in cases(args.configs):
        if cur is not cfg:
            dt = host = None
            torch.cuda.empty_cache()
            cur, dt = cfg, table_for(cfg)
            host = dt.reference_soa()
        item = dt.dtype.itemsize
        S = {"v": 1, "vgl": 5, "vgh": 10}[kind]
        P = p.shape[0]
        c = launch_size(P, S, dt.lanes, item)
        dp = torch.from_numpy(np.ascontiguousarray(p)).cuda()
        out = torch.empty((c, S, dt.lanes), dtype=dt.data.dtype, device="cuda")

        def run():
            for lo in range(0, P, c):
                evaluate(dt, kind, dp[lo: lo + c], out[: min(c, P - lo)], check=False)

        t = timed(run, args.reps)
        # parity on the first launch's outputs: stratified oracle sample
        first = p[:c]
        evaluate(dt, kind, dp[:c], out[:c], check=False)
        sel = stratified_sample(first, dt.grid, n_min=min(2048, len(first)))
        got = out.index_select(0, torch.from_numpy(sel).cuda())[:, :, : dt.n_splines].double().cpu().numpy()
        ref, scale = oracle.eval_f64(kind, host, dt.n_splines, dt.grid.spacings, first[sel])
        tol = 1e-12 if item == 8 else 1e-5
        ok, worst = oracle.tolerance_check(got, ref, scale, tol)
        bpp = bytes_per_position(kind, dt.n_splines, item, 128 // item)
        irreducible = P * S * dt.lanes * item + -(-P // c) * dt.nbytes
        row = {"config": cfg.index, "kind": kind, "positions": P, "n_splines": dt.n_splines, "dtype": cfg.dtype,
               "launch": c, "path": eval_path(dt, kind, c), "seconds": t,
               "orbital_evals_per_s": P * dt.n_splines / t, "algorithmic_gbs": bpp * P / t / 1e9,
               "fraction": bpp * P / t / 1e9 / peak, "frac_irreducible": irreducible / t / 1e9 / peak,
               "oracle_positions": int(sel.size), "max_err_over_tol_scale": worst, "tol": tol, "parity_ok": ok}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del out, dp
    with open(os.path.join(OUT, "report_time.jsonl"), "w") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")


def phase_ncu(args):
    """One launch of each (config, kind), the first launch of phase_time's plan."""
    import torch

    from paper_1611_02665_b200 import evaluate

    cur, dt = None, None
    for cfg, kind, p in cases(args.configs):
        if cur is not cfg:
            dt = None
            torch.cuda.empty_cache()
            cur, dt = cfg, table_for(cfg)
        S = {"v": 1, "vgl": 5, "vgh": 10}[kind]
        c = launch_size(p.shape[0], S, dt.lanes, dt.dtype.itemsize)
        dp = torch.from_numpy(np.ascontiguousarray(p[:c])).cuda()
        evaluate(dt, kind, dp, check=False)
        torch.cuda.synchronize()


NCU = {"gpu__time_duration.sum": "ms", "dram__bytes_read.sum": "dram_read", "dram__bytes_write.sum": "dram_write",
       "lts__t_sector_hit_rate.pct": "l2_hit", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma",
       "l1tex__throughput.avg.pct_of_peak_sustained_elapsed": "l1tex",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64",
       "lts__throughput.avg.pct_of_peak_sustained_elapsed": "lts"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,
         "second": 1e3, "%": 1}


def ncu_rows(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")]
        if not any(k in name for k in ("line_kernel", "eval_tma_kernel", "eval_kernel")):
            continue
        r = {"kernel": name.split("(")[0][:60]}
        for m, key in NCU.items():
            if m in hdr:
                i = hdr.index(m)
                r[key] = float(vals[i].replace(",", "")) * SCALE.get(units[i].strip(), 1.0)
        out.append(r)
    return out


def phase_md(args):
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        peak = float(json.load(f)["hbm_gbs"])
    rows = [json.loads(x) for x in open(args.time)]
    # --ncu: an .ncu-rep, or the rows already extracted from one on the GPU box (.json)
    ncu = (json.load(open(args.ncu)) if args.ncu.endswith(".json") else ncu_rows(args.ncu)) if args.ncu else []
    cpu = {}
    if args.cpu:
        for ln in open(args.cpu):
            if ln.startswith("{"):
                r = json.loads(ln)
                if "f64 oracle" not in r["dtype"]:
                    cpu[(r["config"], r["kind"])] = r
    lines = [f"| cfg | kernel | GPUs | orbital-evals/s | algorithmic GB/s | fraction of {peak:.1f} GB/s | "
             "irreducible fraction | ncu DRAM GB/s | L2 hit % | L2 throughput % | FMA (fp32) / FP64 pipe % | "
             "max err / (tol·Σ\\|w·c\\|) "
             "(oracle positions) | CPU ref orbital-evals/s (cores) |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for i, r in enumerate(rows):
        n = ncu[i] if i < len(ncu) else {}
        n = n if n and n.get("dram_read") == n.get("dram_read") else {}  # nan: ncu could not replay it
        dram = (n["dram_read"] + n["dram_write"]) / (n["ms"] * 1e-3) / 1e9 if n else None
        pipe = n.get("fp64" if r["dtype"] == "f64" else "fma") if n else None
        c = cpu.get((r["config"], r["kind"]))
        cpu_s = f"{c['all_threads']:.3e} ({c['threads']})" if c else "—"
        kname = f"{r['kind'].upper()} ({r['path']}, {r['dtype']}, N={r['n_splines']})"
        lines.append(
            f"| {r['config']} | {kname} | 1 | {r['orbital_evals_per_s']:.3e} | {r['algorithmic_gbs']:,.0f} | "
            f"{r['fraction']:.2f} | {r['frac_irreducible']:.2f} | "
            f"{'%.0f' % dram if dram else '—'} | {'%.1f' % n['l2_hit'] if n else '—'} | "
            f"{'%.1f' % n['lts'] if n.get('lts') is not None else '—'} | "
            f"{'%.1f' % pipe if pipe is not None else '—'} | "
            f"{r['max_err_over_tol_scale']:.3f} ({r['oracle_positions']}) | "
            f"{cpu_s} |")
    # the BASELINE.md section 4 columns
    base = [f"| cfg | kernel | GPUs | orbital-evals/s | algorithmic GB/s | fraction of {peak:.1f} GB/s "
            "(irreducible-bytes fraction) | ncu DRAM GB/s | L2 hit % | max err / Σ\\|w·c\\| | "
            "CPU ref orbital-evals/s (cores) |", "|---|---|---|---|---|---|---|---|---|---|"]
    for i, r in enumerate(rows):
        n = ncu[i] if i < len(ncu) else {}
        n = n if n and n.get("dram_read") == n.get("dram_read") else {}
        dram = (n["dram_read"] + n["dram_write"]) / (n["ms"] * 1e-3) / 1e9 if n else None
        c = cpu.get((r["config"], r["kind"]))
        cpu_s = (f"{c['all_threads']:.2e} ({c['threads']})" + (" fp32 kernels" if r["dtype"] == "f64" else "")) \
            if c else "—"
        base.append(
            f"| {r['config']} | {r['kind'].upper()} ({r['path']} kernel, {r['dtype']}, N={r['n_splines']}) | 1 | "
            f"{r['orbital_evals_per_s']:.3e} | {r['algorithmic_gbs']:,.0f} | {r['fraction']:.2f} "
            f"({r['frac_irreducible']:.2f}) | {'%.0f' % dram if dram else '—'} | "
            f"{'%.1f' % n['l2_hit'] if n else '—'} | {r['max_err_over_tol_scale'] * r['tol']:.1e} "
            f"(tol {r['tol']:.0e}; {r['oracle_positions']} oracle positions) | {cpu_s} |")
    text = ("## BASELINE.md section 4 columns\n\n" + "\n".join(base) + "\n\n## Extended\n\n"
            + "\n".join(lines) + "\n")
    if args.md:
        with open(args.md, "w") as f:
            f.write(text)
    print(text)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--phase", choices=("time", "ncu", "md"), required=True)
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--time", default=os.path.join(OUT, "report_time.jsonl"))
    ap.add_argument("--ncu", default=None)
    ap.add_argument("--cpu", default=None)
    ap.add_argument("--md", default=None)
    args = ap.parse_args()
    args.configs = [int(c) for c in args.configs.split(",")]
    {"time": phase_time, "ncu": phase_ncu, "md": phase_md}[args.phase](args)


if __name__ == "__main__":
    main()

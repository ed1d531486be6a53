#!/usr/bin/env python
"""ncu capture of bench.py's dominant kernel, recorded for the roofline keys.

On the GPU box (under gpurun, one GPU):

    python profiles/ncu_capture.py --tag r02_cfg4 [-- <extra bench.py args>]

1. runs bench.py once without ncu (it must exit 0) and reads the launch key
   (roofline.ncu_key) and kernel path from its JSON line;
2. captures the first launch of that kernel with
   `ncu --set full --clock-control none --import-source on` (the bench's
   correctness-guard launch: the timed launches' exact shape);
3. writes gpurun_out/ncu_record_<tag>.json ({key: record}, the record carrying
   the CUDA source hash bench.py checks) and gpurun_out/<tag>_summary.txt.

Here, after the call:

    python profiles/ncu_capture.py --merge gpurun_out/ncu_record_<tag>.json

merges the records into profiles/ncu_traffic.json (tracked).
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(ROOT, "gpurun_out")

METRICS = {
    "gpu__time_duration.sum": "ncu_time",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "lts_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed": "l1tex_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "cycle/second": 1, "cycle/nsecond": 1e9,
         "cycle/usecond": 1e6, "%": 1}
KERNEL_RE = {"line": "line_kernel", "window": "line_kernel", "tma": "eval_tma_kernel", "generic": "eval_kernel"}


def parse_raw(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    rec = {"kernel_name": vals[hdr.index("Kernel Name")][:160] if "Kernel Name" in hdr else "?"}
    for metric, name in METRICS.items():
        if metric in hdr:
            i = hdr.index(metric)
            v = float(vals[i].replace(",", ""))
            rec[name] = v * SCALE.get(units[i].strip(), 1.0)
    return rec


def capture(tag, extra, replay="kernel"):
    os.makedirs(OUT, exist_ok=True)
    base = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "1", "--warmup", "3", "--no-cpu",
            "--no-e2e", "--no-extra", *extra]
    plain = subprocess.run(base, capture_output=True, text=True, cwd=ROOT)
    if plain.returncode != 0:
        sys.stderr.write(plain.stderr[-3000:])
        raise SystemExit("plain bench run failed: not capturing")
    line = json.loads([ln for ln in plain.stdout.splitlines() if ln.startswith("{")][-1])
    roof = line["roofline"]
    key = roof["ncu_key"]
    path = line["config"].get("path") or line["config"].get("path_v")
    rep = os.path.join(OUT, f"prof_{tag}")
    cmd = ["ncu", "--set", "full", "--clock-control", "none", "--import-source", "on", "-k",
           f"regex:{KERNEL_RE[path]}", "-c", "1", "-o", rep, "-f",
           *(["--replay-mode", "application"] if replay == "application" else []), *base]
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT)
    with open(os.path.join(OUT, f"ncu_{tag}.log"), "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout[-20000:] + r.stderr[-20000:])
    rec = parse_raw(rep + ".ncu-rep")
    rec["dram_bytes_per_launch"] = rec.get("dram_read", 0) + rec.get("dram_write", 0)
    rec.update(source_hash=roof["source_hash"], positions_per_launch=roof["positions_per_launch"],
               algorithmic_bytes_per_position=roof["algorithmic_bytes_per_position"],
               source=f"profiles/ncu_capture.py --tag {tag}: ncu --set full --clock-control none, first "
                      f"{KERNEL_RE[path]} launch of `bench.py {' '.join(extra)}` (the correctness-guard launch, "
                      f"same shape as the timed ones)")
    with open(os.path.join(OUT, f"ncu_record_{tag}.json"), "w") as f:
        json.dump({key: rec}, f, indent=1)
    summ = subprocess.run([sys.executable, os.path.join(HERE, "ncu_summary.py"), rep + ".ncu-rep"],
                          capture_output=True, text=True).stdout
    with open(os.path.join(OUT, f"{tag}_summary.txt"), "w") as f:
        f.write(f"key {key}\n{json.dumps(rec, indent=1)}\n\n{summ}")
    print(json.dumps({key: rec}))


def merge(paths):
    dst = os.path.join(HERE, "ncu_traffic.json")
    try:
        with open(dst) as f:
            db = json.load(f)
    except FileNotFoundError:
        db = {}
    for p in paths:
        with open(p) as f:
            db.update(json.load(f))
    with open(dst, "w") as f:
        json.dump(db, f, indent=1, sort_keys=True)
        f.write("\n")
    print(f"merged {len(paths)} record file(s) into {dst}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag")
    ap.add_argument("--merge", nargs="*")
    ap.add_argument("--replay", default="kernel", choices=("kernel", "application"),
                    help="application: launches whose buffers ncu's kernel replay cannot save (config 5)")
    ap.add_argument("extra", nargs=argparse.REMAINDER)
    a = ap.parse_args()
    if a.merge:
        return merge(a.merge)
    extra = a.extra[1:] if a.extra[:1] == ["--"] else a.extra
    capture(a.tag or "capture", extra, a.replay)


if __name__ == "__main__":
    main()

"""bench.py keeps the driver's JSON-line contract: the reference arm on the
host (runs here, config 1) and the B200 arm on the GPU (config 2, short)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "1"], 300)
    assert d["impl"] == "reference" and d["unit"] == "orbital-evals/s" and d["value"] > 0
    assert d["higher_is_better"] is True and d["n_gpus"] == 1
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_b200_arm_contract():
    d = _run(["--config", "2", "--steps", "2", "--warmup", "3", "--no-cpu"], 900)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 3 and d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["unit"] == "GB/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert r["bound"] and 0 < r["frac_irreducible"] <= r["frac"]
    assert d["kpower"]["value"] > 0 and d["config"]["table_form"] == "bspline"
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert d["config"]["path"] in ("line", "window", "tma", "generic")


def _torchrun(args, port, timeout=900):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--gpus", "2",
           *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    assert r.stdout.rstrip().splitlines()[-1] == lines[0]  # ... and last
    return json.loads(lines[0])


@pytest.mark.gpu
def test_b200_arm_two_ranks():
    """The driver's N>1 launch (torchrun, one rank per GPU, NCCL): two ranks,
    here sharing the test GPU when it has only one (a functional check of the
    barrier / max-over-ranks / rank-0-prints path; bench.py warns that such a
    run is not a measurement).  Default strong scaling: the 64 walkers are
    split over the ranks; the weak figure rides along."""
    d = _torchrun(["--config", "4", "--walkers", "64", "--chunk", "8192", "--steps", "2", "--warmup", "3",
                   "--no-cpu"], 29613)
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "strong"
    assert d["config"]["walkers_per_rank"] == [32, 32] and d["config"]["positions_per_step"] == 64 * 256
    assert d["config"]["parallelism"].startswith("walker-sharded x2")
    assert d["weak"]["positions_per_step"] == 2 * 64 * 256 and d["weak"]["value"] > 0
    assert len(d["clocks_per_rank"]) == 2
    e = d["e2e"]  # whole-job: both ranks' positions over the slower rank's time
    assert e["ranks"] == 2 and e["value"] > 0 and e["h2d_bytes_per_step"] == 64 * 256 * 24


@pytest.mark.gpu
def test_b200_config5_one_rank():
    d = _run(["--config", "5", "--walkers", "256", "--steps", "2", "--warmup", "3", "--no-cpu"], 900)
    assert d["dtype"] == "f64" and d["value"] > 0 and d["n_gpus"] == 1
    assert d["config"]["positions_per_step"] == 256 * 128
    assert sum(d["config"]["positions_by_kind"].values()) == 256 * 128
    assert d["eval"]["value"] > 0 and "gather_overhead_ms_per_step" in d and d["nccl"]["value"] > 0
    assert d["e2e"]["value"] > 0 and d["roofline"]["avg_launch_ms"] > 0


@pytest.mark.gpu
def test_b200_config5_two_ranks():
    """Orbital-sharded over two ranks: PeerGather's IPC buffer on rank 0 and
    the NCCL/gloo gather baseline, eval and gather timed separately."""
    d = _torchrun(["--config", "5", "--walkers", "128", "--steps", "2", "--warmup", "3", "--no-cpu"], 29617)
    assert d["n_gpus"] == 2 and d["config"]["splines_per_rank"] == [2048, 2048]
    assert d["eval"]["value"] > 0 and d["value"] > 0

"""Fused evaluate + gather over peer memory (multi.PeerGather,
spo_eval_lanes): lane-limited stores, and two torchrun ranks writing their
spline slices into rank 0's buffer through a CUDA IPC mapping (the ranks
share the test box's GPU; they only write disjoint lanes)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from paper_1611_02665_b200 import ContractError, DeviceTable, evaluate
from paper_1611_02665_b200.grid import unit_cell_grid

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("pipeline", [True, False])
@pytest.mark.parametrize("dtype,limit", [("f32", 37), ("f32", 64), ("f64", 23)])
def test_lane_limit_stores_only_leading_lanes(pipeline, dtype, limit):
    import torch

    grid = unit_cell_grid(20)
    dt = DeviceTable.random(grid, 96, seed=3) if dtype == "f32" else DeviceTable.normal_f64(grid, 96, seed=3)
    pos = np.random.default_rng(1).random((700, 3))
    want = evaluate(dt, "vgh", pos, pipeline=pipeline)
    tdt = want.dtype
    # offset view into a wider buffer, like a rank's slice of the root's rows
    buf = torch.full((700, 10, 200), 7.0, dtype=tdt, device="cuda")
    off = 8
    evaluate(dt, "vgh", pos, buf[:, :, off:], pipeline=pipeline, lane_limit=limit)
    assert torch.equal(buf[:, :, off:off + limit], want[:, :, :limit])
    assert bool((buf[:, :, :off] == 7.0).all()) and bool((buf[:, :, off + limit:] == 7.0).all())


def test_lane_limit_validation():
    import torch

    dt = DeviceTable.random(unit_cell_grid(16), 64, seed=0)
    pos = np.zeros((4, 3))
    with pytest.raises(ContractError):
        evaluate(dt, "v", pos, lane_limit=10)  # needs out
    out = torch.empty((4, 1, 64), device="cuda")
    with pytest.raises(ContractError):
        evaluate(dt, "v", pos, out, lane_limit=65)
    with pytest.raises(ContractError):
        evaluate(dt, "v", pos, out[:, :, 2:], lane_limit=20)  # misaligned lane offset (8 bytes)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("dtype,n", [("f32", 200), ("f64", 90)])
def test_peer_gather_two_ranks(dtype, n):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.join(ROOT, "scripts", "peer_gather_check.py"), "--dtype", dtype, "--splines", str(n)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    res = json.loads([line for line in r.stdout.splitlines() if line.startswith("{")][-1])
    assert res["peer_bitwise"] and res["world"] == 2


def test_peer_gather_two_ranks_kpower():
    """The fused gather on the k-power form: a dense batch (line kernel) on each
    rank's k-power slice, gathered == the full-N k-power evaluation bitwise."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.join(ROOT, "scripts", "peer_gather_check.py"), "--splines", "256", "--positions", "40000",
           "--kpower", "--reps", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    res = json.loads([line for line in r.stdout.splitlines() if line.startswith("{")][-1])
    assert res["peer_bitwise"] and res["world"] == 2 and res["form"] == "kpower"

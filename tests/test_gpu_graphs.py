"""CUDA-graph replay (graphs.GraphedEvaluator) is bitwise identical to
evaluate() for the generic and the TMA-pipelined kernels, fp32 and fp64."""
import numpy as np
import pytest

from paper_1611_02665_b200 import DeviceTable, DomainError, evaluate
from paper_1611_02665_b200.graphs import GraphedEvaluator
from paper_1611_02665_b200.grid import unit_cell_grid

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("pipeline", [True, False])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_graph_replay_bitwise(pipeline, dtype):
    import torch

    grid = unit_cell_grid(24)
    dt = (DeviceTable.random(grid, 256, seed=4) if dtype == "f32"
          else DeviceTable.normal_f64(grid, 128, seed=4))
    g = GraphedEvaluator(dt, "vgh", 1000, pipeline=pipeline)
    rng = np.random.default_rng(0)
    for _ in range(3):
        pos = rng.random((1000, 3)) * 3.0 - 1.0
        got = g.run(pos).clone()
        want = evaluate(dt, "vgh", pos, pipeline=pipeline)
        assert torch.equal(got, want)
    bad = rng.random((1000, 3))
    bad[7, 2] = np.nan
    with pytest.raises(DomainError):
        g.run(bad, check=True)
    g.run(rng.random((1000, 3)), check=True)  # status is reset by every replay


def test_graph_replay_line_path():
    """A dense batch (line-window kernel: cub sort + records + runs + line
    kernel) captured and replayed bitwise."""
    import torch

    from paper_1611_02665_b200.kernels import eval_path

    dt = DeviceTable.random(unit_cell_grid(8), 256, seed=2)
    assert eval_path(dt, "vgh", 3000) == "line"
    g = GraphedEvaluator(dt, "vgh", 3000)
    rng = np.random.default_rng(3)
    for _ in range(3):
        pos = rng.random((3000, 3))
        assert torch.equal(g.run(pos).clone(), evaluate(dt, "vgh", pos))

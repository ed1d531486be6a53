"""CUDA-graph replay of a fixed-shape evaluation (the launch-bound regime).

A QMC driver evaluates the same table at a new batch of positions every move
(driver.py:213-233 calls eval_batch once per walker and kernel).  Each
evaluate() call costs host work plus up to four launches (workspace reset,
bucketing, records, eval kernel); for small batches that dominates.
GraphedEvaluator captures one evaluate() of a fixed batch size into a CUDA
graph over static position / output buffers; run(positions) copies the new
positions in and replays the graph -- one graph launch per call.  Results
are bitwise identical to evaluate() (same kernels, same inputs).
"""
from __future__ import annotations

from .device import as_device_table
from .errors import ContractError
from .kernels import as_kind, evaluate


class GraphedEvaluator:
    """evaluate(table, kind, positions[P]) captured for a fixed P."""

    def __init__(self, table, kind, n_positions: int, *, mode: str = "fast", pipeline="auto",
                 form: str = "auto"):
        import torch

        self.table = as_device_table(table)
        self.kind = as_kind(kind)
        self.n = int(n_positions)
        if self.n < 1:
            raise ContractError("n_positions must be >= 1")
        dev = self.table.device
        tdt = torch.float64 if self.table.dtype.itemsize == 8 else torch.float32
        self.positions = torch.zeros((self.n, 3), dtype=torch.float64, device=dev)
        self.out = torch.empty((self.n, self.kind.output_streams_soa, self.table.lanes), dtype=tdt, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self._kw = dict(mode=mode, pipeline=pipeline, status=self.status, check=False, form=form)
        # warm up outside capture (library load, attributes, allocator pools)
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            evaluate(self.table, self.kind, self.positions, self.out, **self._kw)
        torch.cuda.current_stream(dev).wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.status.zero_()
            evaluate(self.table, self.kind, self.positions, self.out, **self._kw)

    def run(self, positions, check: bool = False):
        """Copy `positions` (n, 3) into the static buffer and replay; returns
        the static output tensor [n][S][lanes] (overwritten by the next run)."""
        import torch

        pos = torch.as_tensor(positions, dtype=torch.float64, device=self.positions.device)
        if tuple(pos.shape) != (self.n, 3):
            raise ContractError(f"positions must be ({self.n}, 3), got {tuple(pos.shape)}")
        self.positions.copy_(pos, non_blocking=True)
        self.graph.replay()
        if check and int(self.status.item()) != 0:
            from .errors import DomainError

            raise DomainError("positions contain non-finite components")
        return self.out

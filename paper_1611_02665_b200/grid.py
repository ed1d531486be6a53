"""Periodic grid spec and the per-position prologue (reference grid.py).

``GridSpec`` mirrors grid.py:34-81 (same fields, validation and derived
properties).  The numeric helpers -- ``map_to_grid`` (grid.py:155-167),
``basis_weights[_batch]`` (grid.py:180-203) and ``compute_prefactors``
(grid.py:206-213) -- run the bit-exact device prologue (csrc/spo_prologue.cuh)
through the C ABI; there is no host implementation.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from .errors import ConfigError, DomainError


def _is_count(n) -> bool:
    return isinstance(n, (int, np.integer)) and n >= 4


def _is_spacing(d) -> bool:
    return d > 0.0 and math.isfinite(d)


def _require_delta(delta) -> float:
    if not _is_spacing(delta):
        raise DomainError(f"spacing delta must be finite and positive (got {delta!r})")
    return float(delta)


@dataclass(frozen=True)
class GridSpec:
    """A 3D uniform grid with periodic wraparound (grid.py:34-81)."""

    nx: int
    ny: int
    nz: int
    dx: float = 1.0
    dy: float = 1.0
    dz: float = 1.0
    periodic: bool = True

    def __post_init__(self):
        # validation as grid.py:44-58 (same exception types; own wording)
        bad = [f"{a}={getattr(self, a)!r}" for a in ("nx", "ny", "nz") if not _is_count(getattr(self, a))]
        if bad:
            raise ConfigError("grid point counts need integers of at least 4: " + ", ".join(bad))
        bad = [f"{a}={getattr(self, a)!r}" for a in ("dx", "dy", "dz") if not _is_spacing(getattr(self, a))]
        if bad:
            raise ConfigError("grid spacings need finite positive values: " + ", ".join(bad))
        if self.periodic is not True:
            raise ConfigError("GridSpec supports periodic boundaries only")

    counts = property(lambda self: (self.nx, self.ny, self.nz))
    spacings = property(lambda self: (self.dx, self.dy, self.dz))
    lengths = property(lambda self: tuple(n * d for n, d in zip(self.counts, self.spacings)))
    # grid.py:75-77 -- 1/d on the host in fp64, the value the reference passes
    inverse_spacings = property(lambda self: tuple(1.0 / d for d in self.spacings))
    n_points = property(lambda self: self.nx * self.ny * self.nz)

    @property
    def padded_counts(self) -> tuple:
        """Device table extent per axis: n + 3 (wrap padding)."""
        return (self.nx + 3, self.ny + 3, self.nz + 3)


def unit_cell_grid(n: int) -> GridSpec:
    """GridSpec(n, n, n, 1/n, 1/n, 1/n): the BASELINE configs' [0,1)^3 cell."""
    return GridSpec(n, n, n, 1.0 / n, 1.0 / n, 1.0 / n)


@dataclass(frozen=True)
class GridPoint:
    """Lower-bound stencil indices and fractional offsets (grid.py:84-93)."""

    i0: int
    j0: int
    k0: int
    tx: float
    ty: float
    tz: float


@dataclass(frozen=True)
class BasisWeights:
    """Per-axis float32 weights a, da, d2a (grid.py:96-106)."""

    a: np.ndarray
    da: np.ndarray
    d2a: np.ndarray


def _device_prologue(pos: np.ndarray, grid: GridSpec, dtype=np.float32):
    """Run spo_prologue on the device for host positions (P,3) float64."""
    import torch

    from . import _abi

    L = _abi.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    p = torch.from_numpy(np.ascontiguousarray(pos, dtype=np.float64)).to(dev)
    n = p.shape[0]
    idx = torch.empty((n, 3), dtype=torch.int32, device=dev)
    t = torch.empty((n, 3), dtype=torch.float64, device=dev)
    tdt = torch.float32 if dtype == np.float32 else torch.float64
    w = torch.empty((n, 3, 3, 4), dtype=tdt, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    _abi.check(L.spo_prologue(0 if dtype == np.float32 else 1, _abi.i32x3(grid.counts),
                              _abi.f64x3(grid.inverse_spacings), _abi.f64x3(grid.spacings),
                              p.data_ptr(), n, idx.data_ptr(), t.data_ptr(), w.data_ptr(),
                              ctypes.c_void_p(stream)))
    return idx.cpu().numpy(), t.cpu().numpy(), w.cpu().numpy()


def _check_position(pos):
    xyz = (float(pos[0]), float(pos[1]), float(pos[2]))
    if not all(map(math.isfinite, xyz)):
        raise DomainError(f"cannot map a non-finite position {xyz} onto the grid")
    return xyz


def map_to_grid(pos, grid: GridSpec) -> GridPoint:
    """Locate a position on the periodic grid (grid.py:155-167), on the device."""
    x, y, z = _check_position(pos)
    idx, t, _ = _device_prologue(np.array([[x, y, z]]), grid)
    return GridPoint(int(idx[0, 0]), int(idx[0, 1]), int(idx[0, 2]),
                     float(t[0, 0]), float(t[0, 1]), float(t[0, 2]))


def stencil_indices(point: GridPoint, grid: GridSpec) -> np.ndarray:
    """The wrapped 4-point stencil per axis, shape (3, 4) int64 (grid.py:170-177)."""
    out = np.empty((3, 4), dtype=np.int64)
    for row, (i0, n) in enumerate(((point.i0, grid.nx), (point.j0, grid.ny), (point.k0, grid.nz))):
        out[row] = (i0 - 1 + np.arange(4)) % n
    return out


def _weights_at(ts: np.ndarray, delta: float) -> np.ndarray:
    """(len(ts), 3, 4) float32 via spo_basis_weights (grid.py:124-139 bit-exact)."""
    import torch

    from . import _abi

    L = _abi.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    t = torch.from_numpy(np.ascontiguousarray(ts, dtype=np.float64)).to(dev)
    w = torch.empty((t.shape[0], 3, 4), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    _abi.check(L.spo_basis_weights(0, t.data_ptr(), t.shape[0], 1.0 / float(delta), float(delta),
                                   w.data_ptr(), ctypes.c_void_p(stream)))
    return w.cpu().numpy()


def basis_weights(t: float, delta: float = 1.0) -> BasisWeights:
    """Basis weights for an offset t in [0, 1) at spacing delta (grid.py:180-189)."""
    if not 0.0 <= t < 1.0:
        raise DomainError(f"offset t must lie in [0, 1) (got {t!r})")
    w = _weights_at(np.array([float(t)]), _require_delta(delta))[0].copy()
    w.flags.writeable = False
    return BasisWeights(a=w[0], da=w[1], d2a=w[2])


def basis_weights_batch(ts, delta: float = 1.0) -> np.ndarray:
    """Weights for many offsets; (len(ts), 3, 4) float32 (grid.py:192-203)."""
    ts = np.ascontiguousarray(ts, dtype=np.float64)
    if ts.ndim != 1:
        raise DomainError(f"offsets must be a 1-D array (got shape {ts.shape})")
    if np.any(ts < 0.0) or np.any(ts >= 1.0) or np.isnan(ts).any():
        raise DomainError("every offset must lie in [0, 1)")
    delta = _require_delta(delta)
    if not ts.size:
        return np.zeros((0, 3, 4), dtype=np.float32)
    return _weights_at(ts, delta).astype(np.float32)


def compute_prefactors(pos, grid: GridSpec):
    """Grid point plus one BasisWeights per axis (grid.py:206-213)."""
    x, y, z = _check_position(pos)
    idx, t, w = _device_prologue(np.array([[x, y, z]]), grid)
    point = GridPoint(int(idx[0, 0]), int(idx[0, 1]), int(idx[0, 2]),
                      float(t[0, 0]), float(t[0, 1]), float(t[0, 2]))
    weights = []
    for ax in range(3):
        wa = w[0, ax].copy()
        wa.flags.writeable = False
        weights.append(BasisWeights(a=wa[0], da=wa[1], d2a=wa[2]))
    return point, tuple(weights)

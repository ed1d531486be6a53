"""Seeded inputs: the reference's position streams and the BASELINE configs.

``position_stream`` / ``generate_positions`` restate driver.py:174-193: a
counter-based numpy Philox stream with counter [0, walker, iteration,
kernel_id] and key [seed, 0], uniform over the domain (kernel ids V=0, VGL=1,
VGH=2, driver.py:44).  The five BASELINE.json configs are defined on top of
them (SURVEY.md Appendix B records the builder decisions for the parts the
reference does not define: quadrature points and the 12:1:1 call mix).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .grid import GridSpec, unit_cell_grid

KERNEL_STREAM_ID = {"v": 0, "vgl": 1, "vgh": 2}


def position_stream(seed, walker, iteration, kernel_id, ns, grid: GridSpec) -> np.ndarray:
    """driver.py:174-179."""
    counter = np.array([0, walker, iteration, kernel_id], dtype=np.uint64)
    key = np.array([seed % (1 << 64), 0], dtype=np.uint64)
    rng = np.random.Generator(np.random.Philox(counter=counter, key=key))
    return rng.random((ns, 3)) * np.asarray(grid.lengths)


@dataclass
class SampleSet:
    """Per-walker, per-iteration positions, one (ns, 3) array per kernel (driver.py:162-171)."""

    v: np.ndarray
    vgl: np.ndarray
    vgh: np.ndarray

    def for_kind(self, kind) -> np.ndarray:
        return getattr(self, str(getattr(kind, "value", kind)).lower())


def generate_positions(seed, walker, iteration, ns, grid) -> SampleSet:
    """driver.py:182-193."""
    s = {k: position_stream(seed, walker, iteration, kid, ns, grid) for k, kid in KERNEL_STREAM_ID.items()}
    return SampleSet(**s)


def walker_positions(seed, walkers, iteration, kernel: str, ns, grid) -> np.ndarray:
    """Concatenate the `kernel` streams of the given walkers: [len(walkers)*ns, 3]."""
    kid = KERNEL_STREAM_ID[kernel]
    return np.concatenate([position_stream(seed, w, iteration, kid, ns, grid) for w in walkers])


def quadrature_positions(seed, walker, grid, n_ions=32, n_quad=12, radius=0.05) -> np.ndarray:
    """Builder-defined pseudopotential quadrature points:
    ion sites = position_stream(seed, w, 1, 0, n_ions); n_quad unit directions
    per ion = normalised standard normals of Philox(counter=[0,w,2,0],
    key=[seed,0]); r = ion + radius*dir (not wrapped: mapping wraps)."""
    ions = position_stream(seed, walker, 1, 0, n_ions, grid)
    rng = np.random.Generator(np.random.Philox(counter=np.array([0, walker, 2, 0], dtype=np.uint64),
                                               key=np.array([seed % (1 << 64), 0], dtype=np.uint64)))
    d = rng.standard_normal((n_ions, n_quad, 3))
    d /= np.linalg.norm(d, axis=-1, keepdims=True)
    return (ions[:, None, :] + radius * d).reshape(-1, 3)


@dataclass(frozen=True)
class Config:
    """One BASELINE.json config (index 1..5)."""

    index: int
    n_grid: int
    n_splines: int
    dtype: str          # "f32" | "f64"
    walkers: int
    moves: int
    kernel: str         # main kernel of the electron moves
    description: str

    @property
    def grid(self) -> GridSpec:
        return unit_cell_grid(self.n_grid)

    @property
    def n_positions(self) -> int:
        return self.walkers * self.moves


CONFIGS = {
    1: Config(1, 16, 64, "f32", 1, 512, "vgh", "16^3, N=64, 512 positions, V/VGL/VGH"),
    2: Config(2, 48, 512, "f32", 256, 64, "vgh", "48^3, N=512, 256x64 VGH + 256x32x12 quadrature V"),
    3: Config(3, 48, 2048, "f32", 1024, 128, "vgl", "48^3, N=2048, 1024x128 VGL"),
    4: Config(4, 64, 4096, "f32", 4096, 256, "vgh", "64^3, N=4096, 4096x256 VGH"),
    5: Config(5, 48, 4096, "f64", 16384, 128, "mix", "48^3, N=4096 fp64, 16384x128, V:VGL:VGH 12:1:1"),
}


def config_positions(cfg: Config, walkers=None, seed: int = 1) -> dict:
    """{kernel: (P, 3) positions} for a config.

    cfg1: the VGH stream of walker 0, iteration 0 (512 positions) for all kinds.
    cfg2: VGH electron moves + quadrature V points (32 ions x 12 per walker).
    cfg3/4: the config kernel's stream of each walker, iteration 0.
    cfg5: the V stream of each walker; kernel by global position index mod 14
          (0-11 V, 12 VGL, 13 VGH).
    """
    g = cfg.grid
    walkers = range(cfg.walkers) if walkers is None else walkers
    if cfg.index == 1:
        p = position_stream(seed, 0, 0, KERNEL_STREAM_ID["vgh"], 512, g)
        return {"v": p, "vgl": p, "vgh": p}
    if cfg.index == 2:
        return {"vgh": walker_positions(seed, walkers, 0, "vgh", cfg.moves, g),
                "v": np.concatenate([quadrature_positions(seed, w, g) for w in walkers])}
    if cfg.index in (3, 4):
        return {cfg.kernel: walker_positions(seed, walkers, 0, cfg.kernel, cfg.moves, g)}
    allp = walker_positions(seed, walkers, 0, "v", cfg.moves, g)
    first = (walkers[0] if len(walkers) else 0) * cfg.moves
    r = (np.arange(allp.shape[0]) + first) % 14
    return {"v": allp[r < 12], "vgl": allp[r == 12], "vgh": allp[r == 13]}


def bytes_per_position(kind: str, n_splines: int, itemsize: int = 4, quantum: int = 32) -> int:
    """North-star algorithmic bytes per position: 64*Npad*sizeof(coef) +
    S*Npad*sizeof(out), Npad = N rounded up to 128 bytes."""
    npad = ((n_splines + quantum - 1) // quantum) * quantum
    s = {"v": 1, "vgl": 5, "vgh": 10}[kind]
    return 64 * npad * itemsize + s * npad * itemsize


def device_walker_positions(seed, walker0, n_walkers, iteration, kernel: str, ns, grid: GridSpec,
                            device=None, out=None):
    """walker_positions generated on the device (spo_fill_positions),
    bit-identical to the numpy streams: (n_walkers * ns, 3) float64 CUDA tensor."""
    import ctypes

    import torch

    from . import _abi
    from .device import _resolve_device, _stream_ptr

    device = _resolve_device(device)
    if out is None:
        out = torch.empty((n_walkers * ns, 3), dtype=torch.float64, device=device)
    _abi.check(_abi.load().spo_fill_positions(
        ctypes.c_uint64(int(seed) % (1 << 64)), int(walker0), int(n_walkers), int(iteration),
        KERNEL_STREAM_ID[kernel], int(ns), _abi.f64x3(grid.lengths), out.data_ptr(), _stream_ptr(device)))
    return out

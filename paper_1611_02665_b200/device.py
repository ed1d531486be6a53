"""Device-resident coefficient tables in the wrap-padded AoSoA layout.

Layout (include/spo_b200.h): ``data[m][i'][j'][k'][l]`` with i' < nx+3 etc.,
``l < nb`` where nb is the tile width rounded up to 128 bytes (32 fp32 / 16
fp64 lanes), and ``data[m][i'][j'][k'][l] = ref[(i'-1)%nx][(j'-1)%ny][(k'-1)%nz]
[m*tile_size + l]`` (zero in padding lanes).  The stencil of (i0, j0, k0) is
then the 4x4x4 block of rows starting at (i0, j0, k0) with no modulo, which
reproduces the reference's periodic indexing (kernels.py:153-157).

Untiled tables are the M = 1 case (tile_size = N).  Tiled tables are the
paper's AoSoA (coeffs.py:141-158, tile_table 197-210): M physically separate
slices, so a tile-major sweep keeps one slice L2-resident.

A table may also carry its k-power form (``with_kpower()``, spo_b200.h
SPO_TABLE_KPOWER): ``kdata[m][i'][j'][4*k0 + r][l]`` holds the power-basis
coefficients of the z-cubic of cell k0, which the FAST kernels contract with
7 instead of 12 FMAs per row group (VGH: 248 instead of 328 per orbital).  It
is derived from ``data`` on the device and read only by FAST evaluations that
opt in with form="kpower" (its error bound is relative to the cell's
coefficient magnitudes, weaker than the north-star sum|w*c| bound; see
kernels._table_form); everything else reads ``data``.
"""
from __future__ import annotations

import ctypes
import warnings
import weakref

import numpy as np

from . import _abi
from .coeffs import CoeffTableAoS, CoeffTableSoA, TiledCoeffTable, padded_count, spline_keys
from .errors import ConfigError, ContractError
from .grid import GridSpec


def _torch():
    import torch

    return torch


def lane_quantum(dtype) -> int:
    """Lanes per 128-byte row quantum."""
    return 16 if np.dtype(dtype) == np.float64 else 32


def _round_up(n: int, q: int) -> int:
    return ((n + q - 1) // q) * q


# L2 working-set target for one AoSoA tile slice: B200 caches per die (2 x ~63 MB),
# and the next unit plus the output stream share it (measured: 40 MB beats 80 MB).
TILE_SLICE_BYTES = 40 << 20
SPATIAL_BUCKETS = 64  # csrc/spo_eval_tma.cu NBUCKET (4 x 4 x 4 blocks)


def auto_tile_size(grid: GridSpec, n_splines: int, dtype=np.float32):
    """AoSoA tile width (splines): the widest of 512/256/128-byte rows (the
    TMA kernel's chunk widths) whose per-spatial-block slice fits the L2
    working-set target; untiled when N fits in one such tile.  Tiles are
    multiples of the 128-byte lane quantum, so spline n keeps output lane n."""
    rows = int(np.prod(grid.padded_counts))
    item = np.dtype(dtype).itemsize
    q = lane_quantum(dtype)
    tile = q
    # the TMA kernel bins positions into SPATIAL_BUCKETS blocks of the grid:
    # its working set is one block's rows x tile (512, 256 or 128-byte rows)
    for row_bytes in (512, 256, 128):
        cand = row_bytes // item
        if cand % q == 0 and rows * row_bytes // SPATIAL_BUCKETS <= TILE_SLICE_BYTES:
            tile = cand
            break
    if n_splines <= tile:
        return None
    return tile


def _resolve_device(device):
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1611_02665_b200 needs a CUDA device (no CPU fallback)")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    device = torch.device(device)
    if device.type != "cuda":
        raise ContractError(f"device tables live on CUDA devices, got {device}")
    if device.index is None:
        device = torch.device("cuda", torch.cuda.current_device())
    return device


def _stream_ptr(device):
    return ctypes.c_void_p(_torch().cuda.current_stream(device).cuda_stream)


class DeviceTable:
    """An immutable device table: grid, N splines, dtype, tiling and storage."""

    def __init__(self, grid: GridSpec, n_splines: int, dtype, tile_size: int, data):
        self.grid = grid
        self.n_splines = int(n_splines)
        self.dtype = np.dtype(dtype)
        if self.dtype not in (np.float32, np.float64):
            raise ContractError("device tables are float32 or float64")
        self.tile_size = int(tile_size)
        self.n_tiles = (self.n_splines + self.tile_size - 1) // self.tile_size
        self.nb = _round_up(self.tile_size, lane_quantum(self.dtype))
        nxp, nyp, nzp = grid.padded_counts
        shape = (self.n_tiles, nxp, nyp, nzp, self.nb)
        if tuple(data.shape) != shape:
            raise ContractError(f"device data shape {tuple(data.shape)} != {shape}")
        self.data = data
        self.device = data.device
        self.kdata = None  # k-power form (with_kpower)

    # ---------------------------------------------------------- geometry --
    @property
    def lanes(self) -> int:
        """Output lanes per stream: n_tiles * nb (spline n -> lane_of(n))."""
        return self.n_tiles * self.nb

    @property
    def dtype_code(self) -> int:
        return _abi.F64 if self.dtype == np.float64 else _abi.F32

    @property
    def nbytes(self) -> int:
        return self.data.numel() * self.data.element_size()

    @property
    def tiled(self) -> bool:
        return self.n_tiles > 1

    def lane_of(self, n):
        """Output lane of spline n (identity when untiled)."""
        n = np.asarray(n)
        return (n // self.tile_size) * self.nb + n % self.tile_size

    @property
    def lanes_are_splines(self) -> bool:
        """Output lane n holds spline n for every n < N (untiled, or tiles
        without padding lanes): the layout spo_eval_lanes needs."""
        return self.n_tiles == 1 or self.tile_size == self.nb

    def lane_index(self):
        """int64 tensor of the lanes of splines 0..N-1 (for compaction)."""
        torch = _torch()
        return torch.from_numpy(self.lane_of(np.arange(self.n_splines)).astype(np.int64)).to(self.device)

    @staticmethod
    def _shape(grid, n_splines, dtype, tile_size):
        if tile_size == "auto":
            tile_size = auto_tile_size(grid, n_splines, dtype)
        tile_size = int(tile_size or n_splines)
        if tile_size < 1:
            raise ConfigError(f"tile_size={tile_size} must be >= 1")
        n_tiles = (n_splines + tile_size - 1) // tile_size
        nb = _round_up(tile_size, lane_quantum(dtype))
        return tile_size, (n_tiles,) + grid.padded_counts + (nb,)

    # ----------------------------------------------------- construction --
    @classmethod
    def empty(cls, grid, n_splines, dtype=np.float32, tile_size="auto", device=None):
        torch = _torch()
        device = _resolve_device(device)
        tile_size, shape = cls._shape(grid, n_splines, dtype, tile_size)
        tdt = torch.float64 if np.dtype(dtype) == np.float64 else torch.float32
        return cls(grid, n_splines, dtype, tile_size, torch.empty(shape, dtype=tdt, device=device))

    @classmethod
    def from_host(cls, table, tile_size="auto", device=None) -> "DeviceTable":
        """Upload a reference-style host table (CoeffTableSoA / TiledCoeffTable /
        CoeffTableAoS, from this package or from bspb itself)."""
        torch = _torch()
        layout = getattr(table, "layout", None)
        if layout == "aosoa" or isinstance(table, TiledCoeffTable):
            tiles = table.tiles
            data = np.concatenate([np.asarray(t.data)[..., : t.n_splines] for t in tiles], axis=-1)
            n = data.shape[-1]
            src_npad = n
            ts = table.tile_size if tile_size in (None, "auto") else tile_size
        elif layout == "aos" or isinstance(table, CoeffTableAoS):
            data = np.moveaxis(np.asarray(table.data), 0, -1)
            n = table.n_splines
            src_npad = n
            ts = tile_size
        elif layout == "soa" or isinstance(table, CoeffTableSoA):
            data = np.asarray(table.data)
            n = table.n_splines
            src_npad = data.shape[-1]
            ts = tile_size
        else:
            raise ContractError(f"unsupported table type {type(table).__name__}")
        data = np.ascontiguousarray(data)
        if data.dtype not in (np.float32, np.float64):
            raise ContractError("coefficients must be float32 or float64")
        g = table.grid
        grid = g if isinstance(g, GridSpec) else GridSpec(g.nx, g.ny, g.nz, g.dx, g.dy, g.dz)
        dt = cls.empty(grid, n, data.dtype, ts, device)
        with warnings.catch_warnings():  # read-only host tables are only read
            warnings.simplefilter("ignore", UserWarning)
            src = torch.from_numpy(data).to(dt.device)
        _abi.check(_abi.load().spo_pack_table(dt.dtype_code, src.data_ptr(), src_npad, n,
                                              _abi.i32x3(grid.counts), dt.tile_size, dt.nb,
                                              dt.n_tiles, dt.data.data_ptr(), _stream_ptr(dt.device)))
        torch.cuda.current_stream(dt.device).synchronize()  # src is freed on return
        return dt

    @classmethod
    def random(cls, grid, n_splines, seed=0, tile_size="auto", device=None) -> "DeviceTable":
        """FillSpec.random(seed) generated on the device, bit-identical to
        build_table(grid, N, FillSpec.random(seed)) (coeffs.py:80-94, 165-185)."""
        torch = _torch()
        dt = cls.empty(grid, n_splines, np.float32, tile_size, device)
        keys = torch.from_numpy(spline_keys(seed, n_splines).view(np.int64)).to(dt.device)
        _abi.check(_abi.load().spo_fill_uniform(keys.data_ptr(), n_splines, _abi.i32x3(grid.counts),
                                                dt.tile_size, dt.nb, dt.n_tiles, dt.data.data_ptr(),
                                                _stream_ptr(dt.device)))
        torch.cuda.current_stream(dt.device).synchronize()
        return dt

    @classmethod
    def normal_f64(cls, grid, n_splines, seed=0, tile_size="auto", device=None, first_spline=0) -> "DeviceTable":
        """Builder-defined fp64 N(0,1) table (BASELINE config 5; spo_b200.h).
        first_spline > 0 generates splines [first_spline, first_spline +
        n_splines) of the full table directly -- an orbital shard, equal to
        slice_orbitals() of the full table without building it."""
        torch = _torch()
        dt = cls.empty(grid, n_splines, np.float64, tile_size, device)
        keys_np = spline_keys(seed, first_spline + n_splines)[first_spline:]
        keys = torch.from_numpy(np.ascontiguousarray(keys_np).view(np.int64)).to(dt.device)
        _abi.check(_abi.load().spo_fill_normal_f64(keys.data_ptr(), n_splines, _abi.i32x3(grid.counts),
                                                   dt.tile_size, dt.nb, dt.n_tiles, dt.data.data_ptr(),
                                                   _stream_ptr(dt.device)))
        torch.cuda.current_stream(dt.device).synchronize()
        return dt

    # ---------------------------------------------------- k-power form --
    @property
    def kpower_shape(self):
        nx, ny, nz = self.grid.counts
        return (self.n_tiles, nx + 3, ny + 3, 4 * nz, self.nb)

    @property
    def has_kpower(self) -> bool:
        return self.kdata is not None

    def with_kpower(self) -> "DeviceTable":
        """Build (once) the k-power form of this table on its device and
        return self.  Costs 4 nz / (nz + 3) times the table's memory (config
        4: 18.8 GB next to the 4.9 GB B-spline form)."""
        if self.kdata is None:
            torch = _torch()
            kd = torch.empty(self.kpower_shape, dtype=self.data.dtype, device=self.device)
            _abi.check(_abi.load().spo_pack_kpower(self.dtype_code, self.data.data_ptr(),
                                                   _abi.i32x3(self.grid.counts), self.nb, self.n_tiles,
                                                   kd.data_ptr(), _stream_ptr(self.device)))
            torch.cuda.current_stream(self.device).synchronize()
            self.kdata = kd
        return self

    def drop_kpower(self) -> "DeviceTable":
        self.kdata = None
        return self

    def slice_orbitals(self, lo: int, hi: int, tile_size="auto") -> "DeviceTable":
        """A new device table holding splines [lo, hi) (orbital sharding)."""
        ref = self.reference_soa(device_result=True)
        torch = _torch()
        sub = ref[..., lo:hi].contiguous()
        n = hi - lo
        dt = DeviceTable.empty(self.grid, n, self.dtype, tile_size, self.device)
        _abi.check(_abi.load().spo_pack_table(dt.dtype_code, sub.data_ptr(), n, n,
                                              _abi.i32x3(self.grid.counts), dt.tile_size, dt.nb,
                                              dt.n_tiles, dt.data.data_ptr(), _stream_ptr(dt.device)))
        torch.cuda.current_stream(dt.device).synchronize()
        return dt

    def reference_soa(self, device_result: bool = False):
        """The table in the reference SoA layout [nx][ny][nz][npad16] (float32
        or float64), e.g. for the CPU oracle.  Rows i' = 1..n are the
        unwrapped grid; lanes are compacted across tiles."""
        nx, ny, nz = self.grid.counts
        inner = self.data[:, 1: nx + 1, 1: ny + 1, 1: nz + 1, :]
        parts = [inner[m, ..., : min(self.tile_size, self.n_splines - m * self.tile_size)]
                 for m in range(self.n_tiles)]
        torch = _torch()
        full = torch.cat(parts, dim=-1) if len(parts) > 1 else parts[0]
        npad = padded_count(self.n_splines)
        out = torch.zeros((nx, ny, nz, npad), dtype=full.dtype, device=full.device)
        out[..., : self.n_splines] = full
        if device_result:
            return out
        return out.cpu().numpy()

    def __repr__(self) -> str:
        kp = f" + k-power form {self.kdata.numel() * self.kdata.element_size() / 1e9:.3f} GB" if self.has_kpower else ""
        return (f"DeviceTable(grid={self.grid.counts}, N={self.n_splines}, dtype={self.dtype.name}, "
                f"tile_size={self.tile_size}, n_tiles={self.n_tiles}, nb={self.nb}, "
                f"{self.nbytes / 1e9:.3f} GB{kp} on {self.device})")


_UPLOADS: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def as_device_table(table, device=None) -> DeviceTable:
    """DeviceTable passthrough, or upload a host table once (tables are
    immutable, coeffs.py:107, 130) and cache it per (table object, device)."""
    if isinstance(table, DeviceTable):
        return table
    device = _resolve_device(device)
    try:
        per_table = _UPLOADS.setdefault(table, {})
    except TypeError:  # not weak-referenceable
        per_table = {}
    key = (device.type, device.index)
    if key not in per_table:
        per_table[key] = DeviceTable.from_host(table, device=device)
    return per_table[key]

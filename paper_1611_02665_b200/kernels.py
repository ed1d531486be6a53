"""V / VGL / VGH evaluation: the drop-in surface and the batched device API.

Drop-in (same names, signatures, errors and output semantics as the
reference kernels.py):
    KernelKind, WalkerOutputsSoA, WalkerOutputsAoS, eval_batch, eval_v,
    eval_vgl, eval_vgh, eval_tiled, allocate_outputs, collect_streams.
  ``eval_batch(table, kind, positions, out)`` evaluates every position on the
  GPU and -- like kernels.py:353-354 -- leaves the LAST position's streams in
  the caller's host buffers.

Batched (the north-star entry points):
    evaluate(table, kind, positions, out=None, mode="fast") -> [P][S][lanes]
    evaluate_v / evaluate_vgl / evaluate_vgh(table, positions, ...)
  positions: (P, 3) float64 (device tensor, or host array -> copied), output
  a CUDA tensor with one block of S streams per position (reference stream
  order, kernels.py:46-51); ``streams(...)`` turns it into {name: [P, N]}.

There is no CPU path: everything below calls libspo_b200.so (spo_eval).
"""
from __future__ import annotations

import ctypes
import os
import enum
import threading

import numpy as np

from . import _abi
from .coeffs import CoeffTableAoS, CoeffTableSoA, TiledCoeffTable, aligned_zeros, padded_count
from .device import DeviceTable, _resolve_device, _stream_ptr, as_device_table
from .errors import ConfigError, ContractError, DomainError


class KernelKind(enum.Enum):
    """V = value; VGL = value, gradient, Laplacian; VGH = value, gradient, Hessian
    (kernels.py:26-51)."""

    V = "v"
    VGL = "vgl"
    VGH = "vgh"

    @property
    def output_streams_soa(self) -> int:
        return {KernelKind.V: 1, KernelKind.VGL: 5, KernelKind.VGH: 10}[self]

    @property
    def output_streams_aos(self) -> int:
        return {KernelKind.V: 1, KernelKind.VGL: 5, KernelKind.VGH: 13}[self]

    def output_streams(self, layout: str) -> int:
        return self.output_streams_aos if layout == "aos" else self.output_streams_soa

    @property
    def stream_names(self) -> tuple:
        if self is KernelKind.V:
            return ("v",)
        if self is KernelKind.VGL:
            return ("v", "gx", "gy", "gz", "l")
        return ("v", "gx", "gy", "gz", "hxx", "hxy", "hxz", "hyy", "hyz", "hzz")

    @property
    def code(self) -> int:
        return {KernelKind.V: _abi.KIND_V, KernelKind.VGL: _abi.KIND_VGL, KernelKind.VGH: _abi.KIND_VGH}[self]


def as_kind(kind) -> KernelKind:
    """Accept our KernelKind, the reference's (bspb.kernels.KernelKind) or a string."""
    if isinstance(kind, KernelKind):
        return kind
    value = getattr(kind, "value", kind)
    try:
        return KernelKind(str(value).lower())
    except ValueError:
        raise ContractError(f"unknown kernel kind {kind!r}") from None


class WalkerOutputsSoA:
    """Planar output streams v, g[3], l, h[6] of n_padded lanes (kernels.py:54-88)."""

    layout = "soa"

    def __init__(self, n_splines: int):
        npad = padded_count(n_splines)
        self.n_splines = n_splines
        self.n_padded = npad
        self.v = aligned_zeros(npad)
        self.g = aligned_zeros((3, npad))
        self.l = aligned_zeros(npad)
        self.h = aligned_zeros((6, npad))

    @property
    def nbytes(self) -> int:
        return self.v.nbytes + self.g.nbytes + self.l.nbytes + self.h.nbytes

    def streams(self, kind) -> dict:
        kind = as_kind(kind)
        n = self.n_splines
        out = {"v": self.v[:n]}
        if kind is KernelKind.V:
            return out
        out.update(gx=self.g[0, :n], gy=self.g[1, :n], gz=self.g[2, :n])
        if kind is KernelKind.VGL:
            out["l"] = self.l[:n]
            return out
        for row, name in enumerate(("hxx", "hxy", "hxz", "hyy", "hyz", "hzz")):
            out[name] = self.h[row, :n]
        return out

    def _targets(self, kind):
        """Host rows receiving streams 0..S-1 in reference order."""
        kind = as_kind(kind)
        rows = [self.v]
        if kind is not KernelKind.V:
            rows += [self.g[0], self.g[1], self.g[2]]
            rows += [self.l] if kind is KernelKind.VGL else [self.h[r] for r in range(6)]
        return rows


class WalkerOutputsAoS:
    """Interleaved buffers v[N], g[3N], l[N], h[9N] (kernels.py:91-124)."""

    layout = "aos"

    def __init__(self, n_splines: int):
        self.n_splines = n_splines
        self.v = np.zeros(n_splines, dtype=np.float32)
        self.g = np.zeros(3 * n_splines, dtype=np.float32)
        self.l = np.zeros(n_splines, dtype=np.float32)
        self.h = np.zeros(9 * n_splines, dtype=np.float32)

    @property
    def nbytes(self) -> int:
        return self.v.nbytes + self.g.nbytes + self.l.nbytes + self.h.nbytes

    def streams(self, kind) -> dict:
        kind = as_kind(kind)
        out = {"v": self.v.copy()}
        if kind is KernelKind.V:
            return out
        g = self.g.reshape(-1, 3)
        out.update(gx=g[:, 0].copy(), gy=g[:, 1].copy(), gz=g[:, 2].copy())
        if kind is KernelKind.VGL:
            out["l"] = self.l.copy()
            return out
        h = self.h.reshape(-1, 3, 3)
        for name, (r, c) in (("hxx", (0, 0)), ("hxy", (0, 1)), ("hxz", (0, 2)),
                             ("hyy", (1, 1)), ("hyz", (1, 2)), ("hzz", (2, 2))):
            out[name] = h[:, r, c].copy()
        return out

    def store(self, kind, block: np.ndarray, n: int = None) -> None:
        """Scatter one position's [S][>=n] SoA block (spline-indexed) into the
        first n entries of the interleaved buffers -- n = the table's
        n_splines; entries past it are left untouched, as the reference
        kernels write only the table's splines.  The AoS Hessian stores all
        nine entries (kernels.py:342-350)."""
        kind = as_kind(kind)
        n = self.n_splines if n is None else int(n)
        if n > self.n_splines:
            raise ContractError(f"output buffers ({self.n_splines}) shorter than n_splines ({n})")
        self.v[:n] = block[0, :n]
        if kind is KernelKind.V:
            return
        g = self.g[: 3 * n].reshape(n, 3)
        g[:, 0], g[:, 1], g[:, 2] = block[1, :n], block[2, :n], block[3, :n]
        if kind is KernelKind.VGL:
            self.l[:n] = block[4, :n]
            return
        h = self.h[: 9 * n].reshape(n, 3, 3)
        hxx, hxy, hxz, hyy, hyz, hzz = (block[4 + r, :n] for r in range(6))
        h[:, 0, 0], h[:, 0, 1], h[:, 0, 2] = hxx, hxy, hxz
        h[:, 1, 0], h[:, 1, 1], h[:, 1, 2] = hxy, hyy, hyz
        h[:, 2, 0], h[:, 2, 1], h[:, 2, 2] = hxz, hyz, hzz


# ----------------------------------------------------------- batched API --

_MODES = {"fast": _abi.MODE_FAST, "strict": _abi.MODE_STRICT}


def _torch():
    import torch

    return torch


def _positions_tensor(positions, device):
    """(P,3) float64 contiguous CUDA tensor; host input -> copied."""
    torch = _torch()
    if isinstance(positions, torch.Tensor):
        pos = positions
        if pos.dim() == 1:
            pos = pos.reshape(1, 3)
        if pos.dim() != 2 or pos.shape[1] != 3:
            raise ContractError(f"positions must have shape (ns, 3), got {tuple(pos.shape)}")
        if pos.device != device or pos.dtype != torch.float64 or not pos.is_contiguous():
            pos = pos.to(device=device, dtype=torch.float64).contiguous()
        return pos
    arr = _as_positions(positions)
    return torch.from_numpy(arr).to(device)


# positions x lanes from which the TMA-pipelined kernel beats the generic one
# (scripts/micro/small_batch.py: crossover ~2^19 for N = 64 ... 4096)
PIPELINE_MIN_WORK = 1 << 19


def _table_form(dt, kind, mode: str, form: str, P: int, ws_bytes: int):
    """(data tensor, mode flag) of the table form a request runs on.

    "auto" and "bspline" read the B-spline form: its error is bounded by
    1e-5 (fp32) / 1e-12 (fp64) times sum|w*c| per output element for every
    table and position (the north-star metric).  The k-power form is OPT-IN
    (form="kpower"): ~7% faster on dense batches, but its power-basis z-cubic
    is only accurate to tol * (sum|w*c| + sum_ij |wx_i wy_j| * sum_r |q_r| m_r)
    (q = the cell's power-basis coefficients, m_r the z-derivative factors,
    oracle.kpower_scale) -- relative to the coefficient magnitudes, not to
    sum|w*c| alone -- so a table with steep decay along z, or a single spike,
    misses the north-star bound near t_z -> 1 and at basis zeros
    (tests/test_gpu_adversarial.py)."""
    if form not in ("auto", "bspline", "kpower"):
        raise ContractError(f"unknown table form {form!r}")
    if form == "kpower" and mode != "fast":
        raise ContractError("the k-power table form serves FAST evaluations only")
    if form == "kpower" and not dt.has_kpower:
        raise ContractError("the table has no k-power form (DeviceTable.with_kpower())")
    if form == "kpower":
        return dt.kdata, _abi.TABLE_KPOWER
    return dt.data, 0


def evaluate(table, kind, positions, out=None, *, mode: str = "fast", out_index=None,
             status=None, check: bool = True, pipeline="auto", lane_limit=None, form: str = "auto"):
    """Evaluate `kind` at every position; returns out[P][S][lanes] (CUDA).

    table      DeviceTable (or any host table -> uploaded once and cached)
    positions  (P, 3) float64; any finite value (periodic wrap, grid.py:155-167)
    out        optional preallocated CUDA tensor [>=P][S][lanes] of the table dtype
    mode       "fast" (separable FMA) or "strict" (bitwise = reference fp32 kernels)
    out_index  optional int64 CUDA tensor: position p is written to out[out_index[p]]
    status     optional int32 CUDA tensor(1): set to 1 on a non-finite position
    check      raise DomainError for non-finite positions (one sync on status)
    pipeline   fast mode: True = the TMA-pipelined kernels (a workspace is
               allocated here; the line-window kernel for dense batches --
               VGL/VGH >= 1 position per grid cell, V >= 2 -- else the
               per-position kernel),
               False = the generic kernel, "auto" = pipelined when
               P * lanes >= PIPELINE_MIN_WORK.  Same bits either way
               (eval_path() tells which kernel runs)
    lane_limit store only output lanes [0, lane_limit) (spo_eval_lanes); `out`
               is then required and may live on another GPU (a peer
               device's memory or an IPC mapping of it): the fused
               evaluate + gather of multi.PeerGather
    form       "auto" / "bspline": the B-spline table form (the north-star
               error bound for every input); "kpower": the opt-in k-power form
               (DeviceTable.with_kpower) with the weaker bound documented in
               _table_form / DESIGN.md 5.6
    """
    torch = _torch()
    kind = as_kind(kind)
    dt = as_device_table(table)
    device = dt.device
    pos = _positions_tensor(positions, device)
    P = pos.shape[0]
    S = kind.output_streams_soa
    tdt = torch.float64 if dt.dtype == np.float64 else torch.float32
    if lane_limit is not None:
        lane_limit = int(lane_limit)
        if out is None:
            raise ContractError("lane_limit needs a preallocated out tensor")
        if not 1 <= lane_limit <= dt.lanes:
            raise ContractError(f"lane_limit {lane_limit} outside [1, {dt.lanes}]")
        if out.dtype != tdt or not out.is_cuda:
            raise ContractError("out must be a CUDA tensor of the table dtype")
        if out.dim() != 3 or out.shape[1] != S or out.shape[2] < lane_limit or out.stride(2) != 1:
            raise ContractError(f"out must be [P][{S}][>={lane_limit}] with unit lane stride")
        if out_index is None and out.shape[0] < P:
            raise ContractError(f"out holds {out.shape[0]} positions, need {P}")
    elif out is None:
        out = torch.empty((P, S, dt.lanes), dtype=tdt, device=device)
    else:
        if out.dtype != tdt or out.device != device:
            raise ContractError("out must be a CUDA tensor of the table dtype on the table device")
        if out.dim() != 3 or out.shape[1] != S or out.shape[2] < dt.lanes or out.stride(2) != 1:
            raise ContractError(f"out must be [P][{S}][>={dt.lanes}] with unit lane stride")
        if out_index is None and out.shape[0] < P:
            raise ContractError(f"out holds {out.shape[0]} positions, need {P}")
    if mode not in _MODES:
        raise ContractError(f"unknown mode {mode!r}")
    if mode == "strict" and dt.dtype != np.float32:
        raise ContractError("strict mode reproduces the fp32 reference kernels only")
    if status is not None and (status.device != device or status.dtype != torch.int32 or status.numel() < 1):
        raise ContractError("status must be an int32 CUDA tensor on the table device")
    own_status = status is None and check
    if own_status:
        status = torch.zeros(1, dtype=torch.int32, device=device)
    idx_ptr = None
    if out_index is not None:
        if out_index.dtype != torch.int64 or out_index.device != device or out_index.numel() != P:
            raise ContractError("out_index must be an int64 CUDA tensor with one entry per position")
        if not out_index.is_contiguous():
            raise ContractError("out_index must be contiguous")
        idx_ptr = out_index.data_ptr()
    g = dt.grid
    L = _abi.load()
    if pipeline == "auto":  # small batches: one generic launch beats prologue + TMA setup
        pipeline = P * dt.lanes >= PIPELINE_MIN_WORK
    ws_bytes = int(L.spo_eval_workspace_bytes(kind.code, dt.dtype_code, _MODES[mode], P)) if pipeline else 0
    data, flag = _table_form(dt, kind, mode, form, P, ws_bytes)
    ws = torch.empty(max(ws_bytes, 0), dtype=torch.uint8, device=device) if ws_bytes > 0 else None
    head = (kind.code, dt.dtype_code, _MODES[mode] | flag, data.data_ptr(), _abi.i32x3(g.counts), dt.nb,
            dt.n_tiles, _abi.f64x3(g.inverse_spacings), _abi.f64x3(g.spacings), pos.data_ptr(), P,
            out.data_ptr(), out.stride(0), out.stride(1))
    tail = (idx_ptr, status.data_ptr() if status is not None else None,
            ws.data_ptr() if ws is not None else None, max(ws_bytes, 0), _stream_ptr(device))
    if lane_limit is None:
        _abi.check(L.spo_eval(*head, *tail))
    else:
        _abi.check(L.spo_eval_lanes(*head, lane_limit, *tail))
    if own_status and int(status.item()) != 0:
        raise DomainError("positions contain non-finite components")
    return out


_PATHS = {0: "generic", 1: "tma", 2: "line", 3: "window"}


def eval_path(table, kind, n_positions: int, *, mode: str = "fast", pipeline="auto", form: str = "auto") -> str:
    """The kernel evaluate() runs for this request: "generic" (one pass),
    "tma" (per-position TMA pipeline), "line" (planes shared along grid
    lines) or "window" (the line kernel's variant for sparser batches:
    planes shared by the positions of 2 x 2 (j0, k0) cells) -- spo_eval_path;
    all give bitwise identical results on the same table form (eval_form()
    tells which form)."""
    kind = as_kind(kind)
    dt = as_device_table(table)
    L = _abi.load()
    P = int(n_positions)
    if pipeline == "auto":
        pipeline = P * dt.lanes >= PIPELINE_MIN_WORK
    ws = int(L.spo_eval_workspace_bytes(kind.code, dt.dtype_code, _MODES[mode], P)) if pipeline else 0
    _, flag = _table_form(dt, kind, mode, form, P, ws)
    code = L.spo_eval_path(kind.code, dt.dtype_code, _MODES[mode] | flag, _abi.i32x3(dt.grid.counts), dt.nb,
                           dt.n_tiles, P, max(ws, 0))
    if code < 0:
        raise ContractError("bad evaluation request")
    return _PATHS[code]


def eval_form(table, kind, n_positions: int, *, mode: str = "fast", pipeline="auto", form: str = "auto") -> str:
    """The table form evaluate() reads for this request: "bspline" or "kpower"."""
    kind = as_kind(kind)
    dt = as_device_table(table)
    P = int(n_positions)
    if pipeline == "auto":
        pipeline = P * dt.lanes >= PIPELINE_MIN_WORK
    ws = int(_abi.load().spo_eval_workspace_bytes(kind.code, dt.dtype_code, _MODES[mode], P)) if pipeline else 0
    _, flag = _table_form(dt, kind, mode, form, P, ws)
    return "kpower" if flag else "bspline"


def evaluate_v(table, positions, out=None, **kw):
    return evaluate(table, KernelKind.V, positions, out, **kw)


def evaluate_vgl(table, positions, out=None, **kw):
    return evaluate(table, KernelKind.VGL, positions, out, **kw)


def evaluate_vgh(table, positions, out=None, **kw):
    return evaluate(table, KernelKind.VGH, positions, out, **kw)


def evaluate_ratios(table, kind, positions, coef, *, status=None, check: bool = True):
    """Fused consumer epilogue: for every position p
    and stream s, ratios[p, s] = sum_n stream_s(p, n) * coef[p, n], accumulated
    in fp64, without materialising the [P][S][N] outputs -- in QMC, coef[p]
    is the moved electron's column of the inverse Slater matrix and the
    ratios are the determinant ratio and its gradient / Laplacian / Hessian
    numerators.  coef: (P, N) of the table dtype (device or host).  Returns a
    (P, S) float64 CUDA tensor.  Deterministic (fixed-order reduction)."""
    torch = _torch()
    kind = as_kind(kind)
    dt = as_device_table(table)
    device = dt.device
    pos = _positions_tensor(positions, device)
    P = pos.shape[0]
    S = kind.output_streams_soa
    tdt = torch.float64 if dt.dtype == np.float64 else torch.float32
    coef = torch.as_tensor(coef, device=device)
    if coef.dim() != 2 or coef.shape[0] != P or coef.shape[1] != dt.n_splines:
        raise ContractError(f"coef must be (P={P}, N={dt.n_splines}), got {tuple(coef.shape)}")
    if dt.lanes == dt.n_splines and dt.nb == dt.tile_size:  # lane(n) == n: use coef as is
        lanes = coef.to(tdt).contiguous()
    else:
        lanes = torch.zeros((P, dt.lanes), dtype=tdt, device=device)  # output-lane layout, pad lanes 0
        if dt.tiled:
            lanes.index_copy_(1, dt.lane_index(), coef.to(tdt))
        else:
            lanes[:, : dt.n_splines] = coef.to(tdt)
    ratios = torch.empty((P, S), dtype=torch.float64, device=device)
    if P == 0:
        return ratios
    L = _abi.load()
    ws_bytes = int(L.spo_eval_ratios_workspace_bytes(kind.code, dt.dtype_code, dt.nb, dt.n_tiles, P))
    if ws_bytes < 0:
        raise ConfigError("the ratio epilogue needs table rows of a multiple of 512 bytes "
                          f"(tile of {512 // dt.dtype.itemsize} lanes); got nb={dt.nb}")
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=device)
    own_status = status is None and check
    if own_status:
        status = torch.zeros(1, dtype=torch.int32, device=device)
    g = dt.grid
    _abi.check(L.spo_eval_ratios(
        kind.code, dt.dtype_code, dt.data.data_ptr(), _abi.i32x3(g.counts), dt.nb, dt.n_tiles,
        _abi.f64x3(g.inverse_spacings), _abi.f64x3(g.spacings), pos.data_ptr(), P, lanes.data_ptr(),
        lanes.stride(0), ratios.data_ptr(), status.data_ptr() if status is not None else None,
        ws.data_ptr(), ws_bytes, _stream_ptr(device)))
    if own_status and int(status.item()) != 0:
        raise DomainError("positions contain non-finite components")
    return ratios


def streams(result, table, kind) -> dict:
    """{stream name: [P, N] tensor} from an evaluate() result (tile lanes compacted)."""
    kind = as_kind(kind)
    dt = as_device_table(table)
    if dt.tiled:
        sel = result.index_select(2, dt.lane_index())
    else:
        sel = result[:, :, : dt.n_splines]
    return {name: sel[:, s] for s, name in enumerate(kind.stream_names)}


# ----------------------------------------------------------- drop-in API --

def _check_pair(table, out):
    """kernels.py:415-431.  A longer SoA output is accepted; only the table's
    lanes are written (the reference reads past the rows there)."""
    layout = getattr(table, "layout", None)
    if layout == "soa" or isinstance(table, CoeffTableSoA):
        if getattr(out, "layout", None) != "soa":
            raise ContractError("SoA table requires WalkerOutputsSoA")
        if out.n_padded < table.n_padded:
            raise ContractError(
                f"output streams ({out.n_padded}) shorter than table rows ({table.n_padded})")
    elif layout == "aos" or isinstance(table, CoeffTableAoS):
        if getattr(out, "layout", None) != "aos":
            raise ContractError("AoS table requires WalkerOutputsAoS")
        if out.n_splines < table.n_splines:
            raise ContractError(
                f"output buffers ({out.n_splines}) shorter than n_splines ({table.n_splines})")
    elif isinstance(table, DeviceTable):
        pass
    else:
        raise ContractError(f"unsupported table type {type(table).__name__} (tiled: eval_tiled)")


def _as_positions(pos, check_finite: bool = True) -> np.ndarray:
    """kernels.py:434-442: fp64 C-contiguous (ns, 3); (3,) -> (1, 3)."""
    arr = np.ascontiguousarray(pos, dtype=np.float64)
    if arr.ndim == 1:
        arr = arr.reshape(1, 3) if arr.size == 3 else arr
    if arr.ndim != 2 or arr.shape[1] != 3:
        raise ContractError(f"positions must have shape (ns, 3), got {arr.shape}")
    if check_finite and not np.isfinite(arr).all():
        raise DomainError("positions contain non-finite components")
    return arr


# Drop-in path: positions per device pass (2^19 = 2 per cell of a 64^3 grid:
# the line kernel shares more planes), the scratch bytes it may use, and the
# device memory it leaves free.
DROPIN_CHUNK = 1 << 19
DROPIN_SCRATCH_BYTES = 96 << 30
DROPIN_FREE_RESERVE = 16 << 30
# Batches larger than this are checked for non-finite positions on the device
# (the kernels' status flag) instead of by a host pass; either way DomainError
# is raised before the caller's buffers are touched.
HOST_FINITE_CHECK_MAX = 4096


# Host positions above this size are streamed through pinned staging buffers:
# chunk k+1's host->device copy overlaps chunk k's evaluation.
STAGED_MIN_BYTES = 1 << 20
_staging = threading.local()


def _staging_for(device, n_pos: int):
    """Per thread and device: two pinned [n_pos][3] fp64 host buffers, two
    device position buffers and a copy stream (grown on demand, reused)."""
    torch = _torch()
    cache = getattr(_staging, "by_device", None)
    if cache is None:
        cache = _staging.by_device = {}
    key = (device.type, device.index)
    st = cache.get(key)
    if st is None or st["cap"] < n_pos:
        st = {"cap": n_pos,
              "host": [torch.empty((n_pos, 3), dtype=torch.float64).pin_memory() for _ in range(2)],
              "dev": [torch.empty((n_pos, 3), dtype=torch.float64, device=device) for _ in range(2)],
              "copy": torch.cuda.Stream(device),
              "copied": [torch.cuda.Event() for _ in range(2)],
              "used": [torch.cuda.Event() for _ in range(2)]}
        cache[key] = st
    return st


def _eval_last(table, kind, pos: np.ndarray, mode: str):
    """Evaluate all positions on the device; return the last one's [S][lanes]
    block on the host (reference batch semantics, kernels.py:353-354).
    Large batches are streamed: chunk k+1's positions go host -> pinned ->
    device on a copy stream while chunk k evaluates."""
    torch = _torch()
    dt = as_device_table(table)
    S = kind.output_streams_soa
    P = pos.shape[0]
    item = 8 if dt.dtype == np.float64 else 4
    per_pos = S * dt.lanes * item
    # free device memory, counting what torch's caching allocator holds
    # unused (e.g. the previous call's scratch) as free
    free = (torch.cuda.mem_get_info(dt.device)[0] + torch.cuda.memory_reserved(dt.device)
            - torch.cuda.memory_allocated(dt.device))
    budget = min(DROPIN_SCRATCH_BYTES, max(free - DROPIN_FREE_RESERVE, per_pos))
    chunk = max(1, min(P, DROPIN_CHUNK, budget // per_pos))
    if os.environ.get("SPO_DEBUG_DROPIN"):
        print(f"[dropin] P={P} chunk={chunk} free={free / 2**30:.1f} GiB", flush=True)
    tdt = torch.float64 if dt.dtype == np.float64 else torch.float32
    scratch = torch.empty((chunk, S, dt.lanes), dtype=tdt, device=dt.device)
    status = torch.zeros(1, dtype=torch.int32, device=dt.device)
    last = None
    if pos.nbytes < STAGED_MIN_BYTES:
        dpos = torch.from_numpy(pos).to(dt.device)
        for lo in range(0, P, chunk):
            hi = min(P, lo + chunk)
            evaluate(dt, kind, dpos[lo:hi], scratch, mode=mode, status=status, check=False)
            last = hi - lo - 1
    else:
        st = _staging_for(dt.device, chunk)
        compute = torch.cuda.current_stream(dt.device)
        for k, lo in enumerate(range(0, P, chunk)):
            hi, b = min(P, lo + chunk), k & 1
            st["copied"][b].synchronize()          # the pinned half is free again
            host = st["host"][b][: hi - lo]
            host.numpy()[:] = pos[lo:hi]
            with torch.cuda.stream(st["copy"]):
                st["copy"].wait_event(st["used"][b])  # evaluation of chunk k-2 read it
                st["dev"][b][: hi - lo].copy_(host, non_blocking=True)
                st["copied"][b].record(st["copy"])
            compute.wait_event(st["copied"][b])
            evaluate(dt, kind, st["dev"][b][: hi - lo], scratch, mode=mode, status=status, check=False)
            st["used"][b].record(compute)
            last = hi - lo - 1
    block = scratch[last].cpu().numpy()
    if int(status.item()) != 0:
        raise DomainError("positions contain non-finite components")
    if not dt.lanes_are_splines:  # padded tiles: output lane != spline index
        block = block[:, dt.lane_of(np.arange(dt.n_splines))]
    else:
        block = block[:, : dt.n_splines]
    return dt, block


def eval_batch(table, kind, positions, out, *, mode: str = "fast") -> None:
    """Evaluate at every position in order; `out` keeps the last one
    (kernels.py:445-473).  Tiled tables take one WalkerOutputsSoA per tile."""
    kind = as_kind(kind)
    pos = _as_positions(positions, check_finite=np.size(positions) <= 3 * HOST_FINITE_CHECK_MAX)
    layout = getattr(table, "layout", None)
    if layout == "aosoa" or isinstance(table, TiledCoeffTable):
        if len(out) != table.n_tiles:
            raise ContractError(f"{len(out)} output sets for {table.n_tiles} tiles")
        for tile_out in out:
            if getattr(tile_out, "layout", None) != "soa" or tile_out.n_padded < padded_count(table.tile_size):
                raise ContractError("tiled tables need one WalkerOutputsSoA of tile_size per tile")
        if pos.shape[0] == 0:
            return
        dt, block = _eval_last(table, kind, pos, mode)  # block: [S][N], spline-indexed
        ts = table.tile_size
        for m, tile_out in enumerate(out):
            width = min(ts, dt.n_splines - m * ts)
            for s, row in enumerate(tile_out._targets(kind)):
                row[:width] = block[s, m * ts: m * ts + width]
                row[width: padded_count(ts)] = 0.0
        return
    _check_pair(table, out)
    if pos.shape[0] == 0:
        return
    dt, block = _eval_last(table, kind, pos, mode)
    if getattr(out, "layout", None) == "aos":
        out.store(kind, block, dt.n_splines)
        return
    n = dt.n_splines
    width = min(out.n_padded, dt.lanes)
    for s, row in enumerate(out._targets(kind)):
        row[:n] = block[s, :n]
        row[n:width] = 0.0  # padding lanes stay zero (test_kernels.py:181-187)


def eval_v(table, pos, out, **kw) -> None:
    """value of every spline at one position (kernels.py:476-478)."""
    eval_batch(table, KernelKind.V, pos, out, **kw)


def eval_vgl(table, pos, out, **kw) -> None:
    """value, gradient and Laplacian (kernels.py:481-483)."""
    eval_batch(table, KernelKind.VGL, pos, out, **kw)


def eval_vgh(table, pos, out, **kw) -> None:
    """value, gradient and symmetric Hessian (kernels.py:486-488)."""
    eval_batch(table, KernelKind.VGH, pos, out, **kw)


def eval_tiled(tiled, kind, pos, outs, **kw) -> None:
    """Per-tile evaluation; concatenated outputs equal the untiled ones (kernels.py:491-496)."""
    if not (getattr(tiled, "layout", None) == "aosoa" or isinstance(tiled, TiledCoeffTable)):
        raise ContractError("eval_tiled expects a TiledCoeffTable")
    eval_batch(tiled, kind, pos, outs, **kw)


def allocate_outputs(table):
    """Output buffers matching a table's layout (kernels.py:499-507)."""
    layout = getattr(table, "layout", None)
    if layout == "aosoa" or isinstance(table, TiledCoeffTable):
        return [WalkerOutputsSoA(t.n_splines) for t in table.tiles]
    if layout == "soa" or isinstance(table, CoeffTableSoA):
        return WalkerOutputsSoA(table.n_splines)
    if layout == "aos" or isinstance(table, CoeffTableAoS):
        return WalkerOutputsAoS(table.n_splines)
    raise ContractError(f"unsupported table type {type(table).__name__}")


def collect_streams(out, kind) -> dict:
    """{stream name: float32 array of length N}; tile lists concatenated (kernels.py:510-519)."""
    if isinstance(out, (list, tuple)):
        parts = [o.streams(kind) for o in out]
        return {name: np.concatenate([np.asarray(p[name]) for p in parts]) for name in parts[0]}
    return {name: np.array(arr, copy=True) for name, arr in out.streams(kind).items()}

"""ctypes binding of libspo_b200.so (include/spo_b200.h).

The product has no CPU fallback: if the library is missing or CUDA is not
available every entry point raises.  Error codes map to the reference's
exception types (errors.py:4-17).
"""
from __future__ import annotations

import ctypes
import os
import threading

from .errors import ConfigError, ContractError, DomainError

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libspo_b200.so")

KIND_V, KIND_VGL, KIND_VGH = 0, 1, 2
F32, F64 = 0, 1
MODE_FAST, MODE_STRICT = 0, 1
TABLE_KPOWER = 0x100  # OR-ed into the mode: the table is in the k-power form
ABI_VERSION = 6

EXPORTS = ("spo_abi_version", "spo_last_error", "spo_eval", "spo_eval_lanes", "spo_eval_path",
           "spo_eval_workspace_bytes",
           "spo_eval_ratios", "spo_eval_ratios_workspace_bytes", "spo_prologue",
           "spo_basis_weights",
           "spo_pack_table", "spo_pack_kpower",
           "spo_fill_uniform", "spo_fill_normal_f64", "spo_fill_positions")

_lock = threading.Lock()
_lib = None


class SpoCudaError(RuntimeError):
    """CUDA launch/runtime failure inside libspo_b200.so."""


def load(build_if_missing: bool = True):
    """Load (and if needed build) the native library.  No fallback."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        from .build import needs_build

        alt = os.environ.get("SPO_LIB")  # experiments: a variant build of the library
        if alt:
            L = ctypes.CDLL(alt)
            _bind(L)
            _lib = L
            return L
        if needs_build():
            if not build_if_missing:
                raise RuntimeError(f"{LIB_PATH} is missing or stale; run paper_1611_02665_b200.build")
            from .build import build
            build()
        L = ctypes.CDLL(LIB_PATH)
        _bind(L)
        _lib = L
        return L


def _bind(L):
    """Declare the ctypes signatures of include/spo_b200.h and check the ABI version."""
    i32, i64, dbl, vp, ip = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p, ctypes.c_int
    P = ctypes.POINTER
    L.spo_abi_version.restype = ip
    L.spo_last_error.restype = ctypes.c_char_p
    L.spo_eval.restype = ip
    L.spo_eval.argtypes = [ip, ip, ip, vp, P(i32), i32, i32, P(dbl), P(dbl), vp, i64, vp, i64,
                           i64, vp, vp, vp, i64, vp]
    L.spo_eval_lanes.restype = ip
    L.spo_eval_lanes.argtypes = [ip, ip, ip, vp, P(i32), i32, i32, P(dbl), P(dbl), vp, i64, vp, i64,
                                 i64, i64, vp, vp, vp, i64, vp]
    L.spo_eval_path.restype = ip
    L.spo_eval_path.argtypes = [ip, ip, ip, P(i32), i32, i32, i64, i64]
    L.spo_eval_workspace_bytes.restype = i64
    L.spo_eval_workspace_bytes.argtypes = [ip, ip, ip, i64]
    L.spo_eval_ratios_workspace_bytes.restype = i64
    L.spo_eval_ratios_workspace_bytes.argtypes = [ip, ip, i32, i32, i64]
    L.spo_eval_ratios.restype = ip
    L.spo_eval_ratios.argtypes = [ip, ip, vp, P(i32), i32, i32, P(dbl), P(dbl), vp, i64, vp, i64, vp, vp,
                                  vp, i64, vp]
    L.spo_prologue.restype = ip
    L.spo_prologue.argtypes = [ip, P(i32), P(dbl), P(dbl), vp, i64, vp, vp, vp, vp]
    L.spo_basis_weights.restype = ip
    L.spo_basis_weights.argtypes = [ip, vp, i64, dbl, dbl, vp, vp]
    L.spo_pack_table.restype = ip
    L.spo_pack_table.argtypes = [ip, vp, i32, i32, P(i32), i32, i32, i32, vp, vp]
    L.spo_pack_kpower.restype = ip
    L.spo_pack_kpower.argtypes = [ip, vp, P(i32), i32, i32, vp, vp]
    L.spo_fill_uniform.restype = ip
    L.spo_fill_uniform.argtypes = [vp, i32, P(i32), i32, i32, i32, vp, vp]
    L.spo_fill_normal_f64.restype = ip
    L.spo_fill_normal_f64.argtypes = [vp, i32, P(i32), i32, i32, i32, vp, vp]
    u64 = ctypes.c_uint64
    L.spo_fill_positions.restype = ip
    L.spo_fill_positions.argtypes = [u64, i64, i64, u64, u64, i64, P(dbl), vp, vp]
    if L.spo_abi_version() != ABI_VERSION:
        raise RuntimeError("libspo_b200.so ABI version mismatch; rebuild")


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = (load().spo_last_error() or b"").decode(errors="replace")
    if rc == 1:
        raise ContractError(msg)
    if rc == 2:
        raise DomainError(msg)
    if rc == 3:
        raise ConfigError(msg)
    raise SpoCudaError(msg)


def i32x3(v):
    return (ctypes.c_int32 * 3)(*[int(x) for x in v])


def f64x3(v):
    return (ctypes.c_double * 3)(*[float(x) for x in v])

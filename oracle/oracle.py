"""numpy + C (ctypes) restatement of the reference path -- TEST INFRASTRUCTURE ONLY.

See oracle/__init__.py for the import rule.  Kind codes: V=0, VGL=1, VGH=2
with the reference's stream order (kernels.py:46-51).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

__all__ = [
    "KIND_CODES", "STREAMS", "STREAM_NAMES", "map_axis", "weights_f32", "weights_f64",
    "evaluate_f64_np", "lib", "c_map_axis", "c_weights_f32", "c_weights_f64",
    "eval_f32", "eval_f64", "tolerance_check", "host_threads", "kpower_scale",
]

KIND_CODES = {"v": 0, "vgl": 1, "vgh": 2}
STREAMS = {"v": 1, "vgl": 5, "vgh": 10}
STREAM_NAMES = {
    "v": ("v",),
    "vgl": ("v", "gx", "gy", "gz", "l"),
    "vgh": ("v", "gx", "gy", "gz", "hxx", "hxy", "hxz", "hyy", "hyz", "hzz"),
}

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def _kind(kind) -> str:
    k = getattr(kind, "value", kind)
    if isinstance(k, int):
        return ("v", "vgl", "vgh")[k]
    return str(k).lower()


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


# ---------------------------------------------------------------- numpy ----

def map_axis(x, dinv: float, count: float):
    """grid.py:109-121 vectorised.  numpy's float `%` (np.remainder) follows
    CPython's float_rem exactly: fmod, sign fix-up toward the divisor, +0.0."""
    x = np.asarray(x, dtype=np.float64)
    count = float(count)
    length = count / dinv
    u = np.remainder(np.remainder(x, length) * dinv, count)
    u = np.where(u >= count, u - count, u)
    i = u.astype(np.int64)  # u >= 0: truncation == int()
    return i, u - i


def weights_f32(t, dinv: float) -> np.ndarray:
    """grid.py:124-139: fp64 expressions left to right, one fp32 rounding.
    Returns (..., 3, 4) float32 rows a, da, d2a."""
    t = np.asarray(t, dtype=np.float64)
    s = 1.0 - t
    w = np.empty(t.shape + (3, 4), dtype=np.float64)
    w[..., 0, 0] = s * s * s / 6.0
    w[..., 0, 1] = (3.0 * t * t * t - 6.0 * t * t + 4.0) / 6.0
    w[..., 0, 2] = (-3.0 * t * t * t + 3.0 * t * t + 3.0 * t + 1.0) / 6.0
    w[..., 0, 3] = t * t * t / 6.0
    w[..., 1, 0] = -0.5 * s * s * dinv
    w[..., 1, 1] = (1.5 * t * t - 2.0 * t) * dinv
    w[..., 1, 2] = (-1.5 * t * t + t + 0.5) * dinv
    w[..., 1, 3] = 0.5 * t * t * dinv
    w[..., 2, 0] = s * dinv * dinv
    w[..., 2, 1] = (3.0 * t - 2.0) * dinv * dinv
    w[..., 2, 2] = (1.0 - 3.0 * t) * dinv * dinv
    w[..., 2, 3] = t * dinv * dinv
    return w.astype(np.float32)


def weights_f64(t: float, delta: float) -> np.ndarray:
    """oracle.py:20-42 for one scalar t (Python float ** == C pow)."""
    t = float(t)
    s = 1.0 - t
    a = [s ** 3 / 6.0, (3.0 * t ** 3 - 6.0 * t ** 2 + 4.0) / 6.0,
         (-3.0 * t ** 3 + 3.0 * t ** 2 + 3.0 * t + 1.0) / 6.0, t ** 3 / 6.0]
    da = np.array([-3.0 * s ** 2 / 6.0, (9.0 * t ** 2 - 12.0 * t) / 6.0,
                   (-9.0 * t ** 2 + 6.0 * t + 3.0) / 6.0, 3.0 * t ** 2 / 6.0]) / delta
    d2a = np.array([s, 3.0 * t - 2.0, 1.0 - 3.0 * t, t]) / delta ** 2
    return np.stack([np.array(a), da, d2a])


def evaluate_f64_np(kind, data, n_splines, spacings, pos):
    """oracle.py:74-115 in numpy for small cases.  data: reference SoA
    [nx][ny][nz][npad] (f32 or f64).  Returns [P][S][N] float64."""
    kind = _kind(kind)
    nx, ny, nz = data.shape[:3]
    pos = np.atleast_2d(np.asarray(pos, dtype=np.float64))
    out = np.zeros((pos.shape[0], STREAMS[kind], n_splines))
    for q, (x, y, z) in enumerate(pos):
        idx, w = [], []
        for c, cnt, d in ((x, nx, spacings[0]), (y, ny, spacings[1]), (z, nz, spacings[2])):
            i0, t = map_axis(c, 1.0 / d, cnt)
            idx.append((int(i0) - 1 + np.arange(4)) % cnt)
            w.append(weights_f64(float(t), d))
        block = np.asarray(data[np.ix_(*idx)][..., :n_splines], dtype=np.float64)
        (ax, dax, d2ax), (ay, day, d2ay), (az, daz, d2az) = w
        acc = {k: np.zeros(n_splines) for k in STREAM_NAMES["vgh"]}
        for i in range(4):
            for j in range(4):
                for k in range(4):
                    p = block[i, j, k]
                    acc["v"] += ax[i] * ay[j] * az[k] * p
                    acc["gx"] += dax[i] * ay[j] * az[k] * p
                    acc["gy"] += ax[i] * day[j] * az[k] * p
                    acc["gz"] += ax[i] * ay[j] * daz[k] * p
                    acc["hxx"] += d2ax[i] * ay[j] * az[k] * p
                    acc["hxy"] += dax[i] * day[j] * az[k] * p
                    acc["hxz"] += dax[i] * ay[j] * daz[k] * p
                    acc["hyy"] += ax[i] * d2ay[j] * az[k] * p
                    acc["hyz"] += ax[i] * day[j] * daz[k] * p
                    acc["hzz"] += ax[i] * ay[j] * d2az[k] * p
        acc["l"] = acc["hxx"] + acc["hyy"] + acc["hzz"]
        for s, name in enumerate(STREAM_NAMES[kind]):
            out[q, s] = acc[name]
    return out


# -------------------------------------------------------------------- C ----

def lib():
    """Load oracle/liboracle.so, building it with `make` if missing."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = os.path.join(_HERE, "liboracle.so")
    if not os.path.exists(path):
        subprocess.run(["make", "-C", _HERE, "-s"], check=True)
    L = ctypes.CDLL(path)
    i64, dbl, vp, ip = ctypes.c_int64, ctypes.c_double, ctypes.c_void_p, ctypes.c_int
    L.orc_map_axis.argtypes = [dbl, dbl, dbl, ctypes.POINTER(i64), ctypes.POINTER(dbl)]
    L.orc_weights_f32.argtypes = [dbl, dbl, vp]
    L.orc_weights_f64.argtypes = [dbl, dbl, vp]
    L.orc_eval_f32.argtypes = [ip, vp, ip, ip, ip, ip, dbl, dbl, dbl, vp, i64, vp, i64, i64, ip]
    L.orc_eval_f64.argtypes = [ip, vp, ip, ip, ip, ip, ip, ip, dbl, dbl, dbl, vp, i64, vp, vp,
                               i64, i64, ip]
    L.orc_eval_f32.restype = ip
    L.orc_eval_f64.restype = ip
    _LIB = L
    return L


def c_map_axis(x: float, dinv: float, count: float):
    i = ctypes.c_int64()
    t = ctypes.c_double()
    lib().orc_map_axis(float(x), float(dinv), float(count), ctypes.byref(i), ctypes.byref(t))
    return i.value, t.value


def c_weights_f32(t: float, dinv: float) -> np.ndarray:
    w = np.zeros(12, dtype=np.float32)
    lib().orc_weights_f32(float(t), float(dinv), w.ctypes.data)
    return w.reshape(3, 4)


def c_weights_f64(t: float, delta: float) -> np.ndarray:
    w = np.zeros(12, dtype=np.float64)
    lib().orc_weights_f64(float(t), float(delta), w.ctypes.data)
    return w.reshape(3, 4)


def eval_f32(kind, data, spacings, pos, overwrite=False, nthreads=0):
    """Reference fp32 production kernels (bitwise) over the reference SoA
    table `data` [nx][ny][nz][npad] float32.  Returns [P][S][npad] float32, or
    with overwrite=True the reference batch semantics: only the last
    position's [S][npad] result (kernels.py:353-354)."""
    kind = _kind(kind)
    data = np.ascontiguousarray(data, dtype=np.float32)
    pos = np.ascontiguousarray(np.atleast_2d(pos), dtype=np.float64)
    nx, ny, nz, npad = data.shape
    S = STREAMS[kind]
    P = pos.shape[0]
    if overwrite:
        out = np.zeros((S, npad), dtype=np.float32)
        pstride = 0
    else:
        out = np.zeros((P, S, npad), dtype=np.float32)
        pstride = S * npad
    dinv = [1.0 / float(d) for d in spacings]
    rc = lib().orc_eval_f32(KIND_CODES[kind], data.ctypes.data, nx, ny, nz, npad, *dinv,
                            pos.ctypes.data, P, out.ctypes.data, pstride, npad, int(nthreads))
    if rc:
        raise RuntimeError(f"orc_eval_f32 failed ({rc})")
    return out


def eval_f64(kind, data, n_splines, spacings, pos, with_scale=True, nthreads=0):
    """fp64 oracle (oracle.py:74-115) over the reference SoA table.  Returns
    (values [P][S][N] float64, scale [P][S][N] or None)."""
    kind = _kind(kind)
    data = np.ascontiguousarray(data)
    if data.dtype not in (np.float32, np.float64):
        raise TypeError("table data must be float32 or float64")
    pos = np.ascontiguousarray(np.atleast_2d(pos), dtype=np.float64)
    nx, ny, nz, npad = data.shape
    S = STREAMS[kind]
    P = pos.shape[0]
    N = int(n_splines)
    out = np.zeros((P, S, N))
    scale = np.zeros((P, S, N)) if with_scale else None
    rc = lib().orc_eval_f64(KIND_CODES[kind], data.ctypes.data, int(data.dtype == np.float64),
                            nx, ny, nz, npad, N, *[float(d) for d in spacings], pos.ctypes.data,
                            P, out.ctypes.data, scale.ctypes.data if with_scale else None,
                            S * N, N, int(nthreads))
    if rc:
        raise RuntimeError(f"orc_eval_f64 failed ({rc})")
    return out, scale


def tolerance_check(got, ref, scale, tol):
    """North-star parity metric: |got - ref| <= tol * sum|w*c| per element.
    Returns (ok, worst ratio |got-ref| / (tol*scale))."""
    got = np.asarray(got, dtype=np.float64)
    err = np.abs(got - ref)
    bound = tol * scale
    # a zero scale means every contributing coefficient is 0 -> exact 0 expected
    ratio = np.where(bound > 0, err / np.where(bound > 0, bound, 1.0), np.where(err > 0, np.inf, 0.0))
    worst = float(ratio.max()) if ratio.size else 0.0
    return worst <= 1.0, worst


# (x, y, z) derivative orders of the ten VGH streams (reference order)
_ORDERS = {"v": (0, 0, 0), "gx": (1, 0, 0), "gy": (0, 1, 0), "gz": (0, 0, 1), "hxx": (2, 0, 0),
           "hxy": (1, 1, 0), "hxz": (1, 0, 1), "hyy": (0, 2, 0), "hyz": (0, 1, 1), "hzz": (0, 0, 2)}


def kpower_scale(kind, data, n_splines, spacings, pos):
    """Error scale of the OPT-IN k-power table form -- not a
    reference quantity.  The k-power form evaluates each z-cubic in the power
    basis q0 + q1 t + q2 t^2 + q3 t^3 (q = the basis change of the cell's four
    z coefficients, grid.py:127-130), so its rounding error is relative to
    sum_r |q_r| (times the derivative factors r, r(r-1) and 1/dz, 1/dz^2 for
    z-derivative streams), contracted with |x weights| * |y weights|:

        scale_s = sum_ij |wx_s[i] wy_s[j]| * sum_r |q_r(i, j)| m_s[r],
        m = (1,1,1,1), (0,1,2,3)/dz, (0,0,2,6)/dz^2 for z-order 0, 1, 2;

    VGL `l` takes the three-term sum, as the north-star scale does.  Returns
    [P][S][N] float64.  (The north-star scale sum|w*c| can be far smaller than
    this: a spike at k0-1 has w = (1-t)^3/6 -> 0 as t -> 1 while |q| stays ~1.)"""
    kind = _kind(kind)
    data = np.asarray(data)
    nx, ny, nz = data.shape[:3]
    pos = np.atleast_2d(np.asarray(pos, dtype=np.float64))
    N = int(n_splines)
    dz = float(spacings[2])
    m = (np.array([1.0, 1.0, 1.0, 1.0]), np.array([0.0, 1.0, 2.0, 3.0]) / dz,
         np.array([0.0, 0.0, 2.0, 6.0]) / dz ** 2)
    names = STREAM_NAMES["vgh"]
    out = np.zeros((pos.shape[0], STREAMS[kind], N))
    for q, (x, y, z) in enumerate(pos):
        idx, w = [], []
        for c, cnt, d in ((x, nx, spacings[0]), (y, ny, spacings[1]), (z, nz, spacings[2])):
            i0, t = map_axis(c, 1.0 / d, cnt)
            idx.append((int(i0) - 1 + np.arange(4)) % cnt)
            w.append(np.abs(weights_f64(float(t), d)))
        c = np.asarray(data[np.ix_(*idx)][..., :N], dtype=np.float64)  # [4][4][4][N]
        c0, c1, c2, c3 = (c[:, :, r] for r in range(4))
        qa = np.abs(np.stack([(c0 + 4.0 * c1 + c2) / 6.0, (c2 - c0) / 2.0, (c0 - 2.0 * c1 + c2) / 2.0,
                              ((c3 - c0) + 3.0 * (c1 - c2)) / 6.0]))  # [r][4][4][N]
        acc = {}
        for name in names:
            ox, oy, oz = _ORDERS[name]
            z_mag = np.tensordot(m[oz], qa, axes=(0, 0))  # [4][4][N]
            acc[name] = np.einsum("i,j,ijn->n", w[0][ox], w[1][oy], z_mag)
        acc["l"] = acc["hxx"] + acc["hyy"] + acc["hzz"]
        for s, name in enumerate(STREAM_NAMES[kind]):
            out[q, s] = acc[name]
    return out

// spo_prologue.cuh -- per-position prologue, bit-exact with the reference.
//
// map_axis      grid.py:109-121 (_map_axis) with CPython float `%` semantics
//               (fmod, sign fix-up toward the divisor, +0.0 for a zero
//               remainder).  Every operation is an explicit round-to-nearest
//               intrinsic so no FMA contraction can change a bit.
// weights_f32   grid.py:124-139 (_fill_axis_weights): the fp64 expressions
//               evaluated left to right exactly as written, one rounding to fp32.
// weights_f64   oracle.py:20-42 (axis_weights_f64) form for the fp64 path.
#pragma once
#include <cstdint>

namespace spo {

// CPython float_rem for a positive divisor.
__device__ __forceinline__ double py_mod_pos(double x, double w) {
    double m = fmod(x, w);  // exact (IEEE remainder-type op, 0 ulp)
    if (m != 0.0) {
        if (m < 0.0) m = __dadd_rn(m, w);
    } else {
        m = 0.0;  // copysign(0.0, w) with w > 0
    }
    return m;
}

// grid.py:109-121.  Returns i0 in [0, count); *t in [0, 1).  Non-finite x
// gives NaN t (callers flag it).
__device__ __forceinline__ int map_axis(double x, double dinv, double count, double *t) {
    const double length = __ddiv_rn(count, dinv);
    double u = py_mod_pos(__dmul_rn(py_mod_pos(x, length), dinv), count);
    if (u >= count) u = __dsub_rn(u, count);
    int i = (int)u;  // u >= 0 -> truncation == Python int()
    if (!(u == u)) i = 0;
    *t = __dsub_rn(u, (double)i);
    return i;
}

// grid.py:124-139, w[0..3] = a, w[4..7] = da (x dinv), w[8..11] = d2a (x dinv^2)
__device__ __forceinline__ void weights_f32(double t, double dinv, float *w) {
    const double s = __dsub_rn(1.0, t);
    // s * s * s / 6.0
    w[0] = __double2float_rn(__ddiv_rn(__dmul_rn(__dmul_rn(s, s), s), 6.0));
    // (3.0 * t * t * t - 6.0 * t * t + 4.0) / 6.0
    w[1] = __double2float_rn(__ddiv_rn(
        __dadd_rn(__dsub_rn(__dmul_rn(__dmul_rn(__dmul_rn(3.0, t), t), t),
                            __dmul_rn(__dmul_rn(6.0, t), t)),
                  4.0),
        6.0));
    // (-3.0 * t * t * t + 3.0 * t * t + 3.0 * t + 1.0) / 6.0
    w[2] = __double2float_rn(__ddiv_rn(
        __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(__dmul_rn(-3.0, t), t), t),
                                      __dmul_rn(__dmul_rn(3.0, t), t)),
                            __dmul_rn(3.0, t)),
                  1.0),
        6.0));
    // t * t * t / 6.0
    w[3] = __double2float_rn(__ddiv_rn(__dmul_rn(__dmul_rn(t, t), t), 6.0));
    // -0.5 * s * s * dinv
    w[4] = __double2float_rn(__dmul_rn(__dmul_rn(__dmul_rn(-0.5, s), s), dinv));
    // (1.5 * t * t - 2.0 * t) * dinv
    w[5] = __double2float_rn(
        __dmul_rn(__dsub_rn(__dmul_rn(__dmul_rn(1.5, t), t), __dmul_rn(2.0, t)), dinv));
    // (-1.5 * t * t + t + 0.5) * dinv
    w[6] = __double2float_rn(
        __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(-1.5, t), t), t), 0.5), dinv));
    // 0.5 * t * t * dinv
    w[7] = __double2float_rn(__dmul_rn(__dmul_rn(__dmul_rn(0.5, t), t), dinv));
    // s * dinv * dinv
    w[8] = __double2float_rn(__dmul_rn(__dmul_rn(s, dinv), dinv));
    // (3.0 * t - 2.0) * dinv * dinv
    w[9] = __double2float_rn(__dmul_rn(__dmul_rn(__dsub_rn(__dmul_rn(3.0, t), 2.0), dinv), dinv));
    // (1.0 - 3.0 * t) * dinv * dinv
    w[10] = __double2float_rn(__dmul_rn(__dmul_rn(__dsub_rn(1.0, __dmul_rn(3.0, t)), dinv), dinv));
    // t * dinv * dinv
    w[11] = __double2float_rn(__dmul_rn(__dmul_rn(t, dinv), dinv));
}

// oracle.py:20-42 (fp64, never rounded).  pow(t, 3) is written t*t*t; the
// fp64 path is checked against the oracle at 1e-12 * sum|w*c|, not bitwise.
__device__ __forceinline__ void weights_f64(double t, double delta, double *w) {
    const double s = 1.0 - t;
    const double t2 = t * t, t3 = t2 * t, s2 = s * s;
    w[0] = s2 * s / 6.0;
    w[1] = (3.0 * t3 - 6.0 * t2 + 4.0) / 6.0;
    w[2] = (-3.0 * t3 + 3.0 * t2 + 3.0 * t + 1.0) / 6.0;
    w[3] = t3 / 6.0;
    w[4] = (-3.0 * s2 / 6.0) / delta;
    w[5] = ((9.0 * t2 - 12.0 * t) / 6.0) / delta;
    w[6] = ((-9.0 * t2 + 6.0 * t + 3.0) / 6.0) / delta;
    w[7] = (3.0 * t2 / 6.0) / delta;
    const double d2 = delta * delta;
    w[8] = s / d2;
    w[9] = (3.0 * t - 2.0) / d2;
    w[10] = (1.0 - 3.0 * t) / d2;
    w[11] = t / d2;
}

template <typename T>
__device__ __forceinline__ void axis_weights(double t, double dinv, double delta, T *w);
template <>
__device__ __forceinline__ void axis_weights<float>(double t, double dinv, double, float *w) {
    weights_f32(t, dinv, w);
}
template <>
__device__ __forceinline__ void axis_weights<double>(double t, double, double delta, double *w) {
    weights_f64(t, delta, w);
}

struct GridArgs {
    double dinv[3];
    double cnt[3];
    double delta[3];
    int n[3];
};

}  // namespace spo

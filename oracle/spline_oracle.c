/*
 * spline_oracle.c -- CPU restatement of the reference's tricubic B-spline
 * SPO path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg may load this library, and only as the checker or
 * the CPU baseline -- never as the thing measured or shipped.  The product
 * (paper_1611_02665_b200) never links it.
 *
 * What is restated (reference = /root/reference/pkg/src/bspb):
 *   orc_map_axis      grid.py:109-121 (_map_axis), Python float `%` semantics
 *                     (CPython float_rem: fmod + sign fix-up, +0.0 on zero)
 *   orc_weights_f32   grid.py:124-139 (_fill_axis_weights): fp64 math written
 *                     left to right, no contraction, one rounding to fp32
 *   orc_weights_f64   oracle.py:20-42 (axis_weights_f64): fp64, `**` = pow()
 *   orc_eval_f32      kernels.py:132-247 (_prep, _v_soa, _vgl_soa, _vgh_soa)
 *                     + kernels.py:357-381 (_batch_*_soa): fp32 prefactors
 *                     (a_i*a_j)*a_k, acc += pre*c as separate fp32 mul/add,
 *                     loop order i, j, k, n.  Bitwise equal to the numba
 *                     kernels (pinned by tests/golden, see make_golden.py).
 *   orc_eval_f64      oracle.py:74-115 (evaluate_f64): fp64 weights, block
 *                     upcast, 10-stream fp64 accumulation, VGL l = hxx+hyy+hzz;
 *                     optionally also the per-element tolerance scale
 *                     sum_ijk |W_s(i,j,k) * c| (BASELINE.json north_star).
 *
 * Table layout is the reference SoA layout: data[nx][ny][nz][npad] with
 * periodic wrap by `%` (kernels.py:153-158), NOT the device wrap-padded one.
 *
 * Build: see oracle/Makefile (-O3 -ffp-contract=off -fno-fast-math -fopenmp).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_V 0
#define ORC_VGL 1
#define ORC_VGH 2

static const int kStreams[3] = {1, 5, 10};

/* CPython float_rem (Objects/floatobject.c) for w > 0. */
static double py_mod(double x, double w) {
    double m = fmod(x, w);
    if (m != 0.0) {
        if ((w < 0.0) != (m < 0.0)) m += w;
    } else {
        m = copysign(0.0, w);
    }
    return m;
}

/* grid.py:109-121 */
int orc_map_axis(double x, double dinv, double count, int64_t *i0, double *t) {
    double length = count / dinv;
    double u = py_mod(py_mod(x, length) * dinv, count);
    if (u >= count) u -= count;
    int64_t i = (int64_t)u;
    *i0 = i;
    *t = u - (double)i;
    return 0;
}

/* grid.py:124-139; w = [a0..a3, da0..da3, d2a0..d2a3] */
void orc_weights_f32(double t, double dinv, float *w) {
    double s = 1.0 - t;
    w[0] = (float)(s * s * s / 6.0);
    w[1] = (float)((3.0 * t * t * t - 6.0 * t * t + 4.0) / 6.0);
    w[2] = (float)((-3.0 * t * t * t + 3.0 * t * t + 3.0 * t + 1.0) / 6.0);
    w[3] = (float)(t * t * t / 6.0);
    w[4] = (float)(-0.5 * s * s * dinv);
    w[5] = (float)((1.5 * t * t - 2.0 * t) * dinv);
    w[6] = (float)((-1.5 * t * t + t + 0.5) * dinv);
    w[7] = (float)(0.5 * t * t * dinv);
    w[8] = (float)(s * dinv * dinv);
    w[9] = (float)((3.0 * t - 2.0) * dinv * dinv);
    w[10] = (float)((1.0 - 3.0 * t) * dinv * dinv);
    w[11] = (float)(t * dinv * dinv);
}

/* oracle.py:20-42 (Python `x ** k` on floats is C pow()). */
void orc_weights_f64(double t, double delta, double *w) {
    double s = 1.0 - t;
    w[0] = pow(s, 3.0) / 6.0;
    w[1] = (3.0 * pow(t, 3.0) - 6.0 * pow(t, 2.0) + 4.0) / 6.0;
    w[2] = (-3.0 * pow(t, 3.0) + 3.0 * pow(t, 2.0) + 3.0 * t + 1.0) / 6.0;
    w[3] = pow(t, 3.0) / 6.0;
    w[4] = (-3.0 * pow(s, 2.0) / 6.0) / delta;
    w[5] = ((9.0 * pow(t, 2.0) - 12.0 * t) / 6.0) / delta;
    w[6] = ((-9.0 * pow(t, 2.0) + 6.0 * t + 3.0) / 6.0) / delta;
    w[7] = (3.0 * pow(t, 2.0) / 6.0) / delta;
    double d2 = pow(delta, 2.0);
    w[8] = s / d2;
    w[9] = (3.0 * t - 2.0) / d2;
    w[10] = (1.0 - 3.0 * t) / d2;
    w[11] = t / d2;
}

/* ---- fp32 production-kernel restatement (kernels.py:143-247) ---------- */

/* One position; out streams at out + s*sstride, n in [0, npad). */
#if defined(__x86_64__) && defined(__GNUC__) && !defined(__clang__)
__attribute__((target_clones("avx512f", "avx2", "default")))
#endif
static void eval_one_f32(int kind, const float *data, int nx, int ny, int nz, int npad,
                         double dxi, double dyi, double dzi, const double *p,
                         float *out, int64_t sstride) {
    int64_t i0, j0, k0;
    double tx, ty, tz;
    float wx[12], wy[12], wz[12];
    orc_map_axis(p[0], dxi, (double)nx, &i0, &tx);
    orc_map_axis(p[1], dyi, (double)ny, &j0, &ty);
    orc_map_axis(p[2], dzi, (double)nz, &k0, &tz);
    orc_weights_f32(tx, dxi, wx);
    orc_weights_f32(ty, dyi, wy);
    orc_weights_f32(tz, dzi, wz);
    const float *ax = wx, *dax = wx + 4, *d2ax = wx + 8;
    const float *ay = wy, *day = wy + 4, *d2ay = wy + 8;
    const float *az = wz, *daz = wz + 4, *d2az = wz + 8;
    int S = kStreams[kind];
    for (int s = 0; s < S; ++s) memset(out + s * sstride, 0, sizeof(float) * (size_t)npad);
    float *restrict v = out;
    float *restrict gx = out + 1 * sstride, *restrict gy = out + 2 * sstride,
                    *restrict gz = out + 3 * sstride;
    for (int i = 0; i < 4; ++i) {
        int64_t ii = (i0 - 1 + i + nx) % nx;
        for (int j = 0; j < 4; ++j) {
            int64_t jj = (j0 - 1 + j + ny) % ny;
            for (int k = 0; k < 4; ++k) {
                int64_t kk = (k0 - 1 + k + nz) % nz;
                const float *restrict row = data + ((ii * ny + jj) * nz + kk) * (int64_t)npad;
                float pv = ax[i] * ay[j] * az[k];
                if (kind == ORC_V) {
#pragma omp simd
                    for (int n = 0; n < npad; ++n) v[n] += pv * row[n];
                    continue;
                }
                float pgx = dax[i] * ay[j] * az[k];
                float pgy = ax[i] * day[j] * az[k];
                float pgz = ax[i] * ay[j] * daz[k];
                if (kind == ORC_VGL) {
                    float pl = d2ax[i] * ay[j] * az[k] + ax[i] * d2ay[j] * az[k] +
                               ax[i] * ay[j] * d2az[k];
                    float *restrict l = out + 4 * sstride;
                    /* the streams and the row never alias: let GCC vectorise
                       (too many pointer pairs for its runtime alias checks) */
#pragma omp simd
                    for (int n = 0; n < npad; ++n) {
                        float c = row[n];
                        v[n] += pv * c;
                        gx[n] += pgx * c;
                        gy[n] += pgy * c;
                        gz[n] += pgz * c;
                        l[n] += pl * c;
                    }
                    continue;
                }
                float phxx = d2ax[i] * ay[j] * az[k];
                float phxy = dax[i] * day[j] * az[k];
                float phxz = dax[i] * ay[j] * daz[k];
                float phyy = ax[i] * d2ay[j] * az[k];
                float phyz = ax[i] * day[j] * daz[k];
                float phzz = ax[i] * ay[j] * d2az[k];
                float *restrict hxx = out + 4 * sstride, *restrict hxy = out + 5 * sstride,
                                *restrict hxz = out + 6 * sstride, *restrict hyy = out + 7 * sstride,
                                *restrict hyz = out + 8 * sstride, *restrict hzz = out + 9 * sstride;
#pragma omp simd
                for (int n = 0; n < npad; ++n) {
                    float c = row[n];
                    v[n] += pv * c;
                    gx[n] += pgx * c;
                    gy[n] += pgy * c;
                    gz[n] += pgz * c;
                    hxx[n] += phxx * c;
                    hxy[n] += phxy * c;
                    hxz[n] += phxz * c;
                    hyy[n] += phyy * c;
                    hyz[n] += phyz * c;
                    hzz[n] += phzz * c;
                }
            }
        }
    }
}

/*
 * Evaluate P positions.  out_pos_stride > 0: position p's streams start at
 * out + p*out_pos_stride.  out_pos_stride == 0: reference batch semantics
 * (kernels.py:353-354) -- each worker overwrites a private buffer and only
 * the last position's result lands in `out`.  nthreads <= 0: all cores.
 */
int orc_eval_f32(int kind, const float *data, int nx, int ny, int nz, int npad,
                 double dxi, double dyi, double dzi, const double *pos, int64_t P,
                 float *out, int64_t out_pos_stride, int64_t out_stream_stride, int nthreads) {
    if (kind < 0 || kind > 2) return 1;
    if (P <= 0) return 0;
    int S = kStreams[kind];
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#else
    nthreads = 1;
#endif
    if (out_pos_stride > 0) {
#pragma omp parallel for num_threads(nthreads) schedule(static)
        for (int64_t p = 0; p < P; ++p)
            eval_one_f32(kind, data, nx, ny, nz, npad, dxi, dyi, dzi, pos + 3 * p,
                         out + p * out_pos_stride, out_stream_stride);
        return 0;
    }
    int err = 0;
#pragma omp parallel num_threads(nthreads)
    {
        int tid = 0, nt = 1;
#ifdef _OPENMP
        tid = omp_get_thread_num();
        nt = omp_get_num_threads();
#endif
        float *buf = (float *)aligned_alloc(64, sizeof(float) * (size_t)S * (size_t)npad + 64);
        if (!buf) {
#pragma omp atomic write
            err = 2;
        } else {
            int64_t lo = P * tid / nt, hi = P * (tid + 1) / nt;
            for (int64_t p = lo; p < hi; ++p)
                eval_one_f32(kind, data, nx, ny, nz, npad, dxi, dyi, dzi, pos + 3 * p, buf, npad);
            if (hi == P && hi > lo)
                for (int s = 0; s < S; ++s)
                    memcpy(out + s * out_stream_stride, buf + (size_t)s * npad,
                           sizeof(float) * (size_t)npad);
            free(buf);
        }
    }
    return err;
}

/* ---- fp64 oracle restatement (oracle.py:74-115) ------------------------ */

/*
 * data: SoA [nx][ny][nz][npad] of float32 (data_is_f64 == 0) or float64.
 * Outputs: for stream s of kind (V:1, VGL:5, VGH:10 in reference order),
 * out[p*pos_stride + s*stream_stride + n] for n < n_splines; if scale != NULL
 * the same layout receives sum_ijk |W_s(i,j,k)| * |c| (for VGL `l` the
 * three-term bound sum (|d2x ay az| + |ax d2y az| + |ax ay d2z|) |c|).
 */
int orc_eval_f64(int kind, const void *data, int data_is_f64, int nx, int ny, int nz,
                 int npad, int n_splines, double dx, double dy, double dz, const double *pos,
                 int64_t P, double *out, double *scale, int64_t pos_stride,
                 int64_t stream_stride, int nthreads) {
    if (kind < 0 || kind > 2) return 1;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#else
    nthreads = 1;
#endif
    const int N = n_splines;
    int err = 0;
#pragma omp parallel num_threads(nthreads)
    {
        double *acc = (double *)calloc((size_t)20 * (size_t)N, sizeof(double));
        double *p = (double *)malloc(sizeof(double) * (size_t)N);
        if (!acc || !p) {
#pragma omp atomic write
            err = 2;
        } else {
#pragma omp for schedule(dynamic, 1)
            for (int64_t q = 0; q < P; ++q) {
                const double *r = pos + 3 * q;
                int64_t i0, j0, k0;
                double tx, ty, tz, wx[12], wy[12], wz[12];
                /* oracle.py:79-81: dinv = 1.0 / grid.dx, integer count */
                orc_map_axis(r[0], 1.0 / dx, (double)nx, &i0, &tx);
                orc_map_axis(r[1], 1.0 / dy, (double)ny, &j0, &ty);
                orc_map_axis(r[2], 1.0 / dz, (double)nz, &k0, &tz);
                orc_weights_f64(tx, dx, wx);
                orc_weights_f64(ty, dy, wy);
                orc_weights_f64(tz, dz, wz);
                memset(acc, 0, sizeof(double) * (size_t)20 * (size_t)N);
                double *A = acc, *B = acc + (size_t)10 * N; /* values, scales */
                for (int i = 0; i < 4; ++i) {
                    int64_t ii = (i0 - 1 + i + nx) % nx;
                    for (int j = 0; j < 4; ++j) {
                        int64_t jj = (j0 - 1 + j + ny) % ny;
                        for (int k = 0; k < 4; ++k) {
                            int64_t kk = (k0 - 1 + k + nz) % nz;
                            int64_t off = ((ii * ny + jj) * nz + kk) * (int64_t)npad;
                            if (data_is_f64) {
                                memcpy(p, (const double *)data + off, sizeof(double) * (size_t)N);
                            } else {
                                const float *f = (const float *)data + off;
                                for (int n = 0; n < N; ++n) p[n] = (double)f[n];
                            }
                            /* prefactor order matches `ax[i] * ay[j] * az[k] * p` */
                            double pre[10] = {
                                wx[i] * wy[j] * wz[k],         wx[4 + i] * wy[j] * wz[k],
                                wx[i] * wy[4 + j] * wz[k],     wx[i] * wy[j] * wz[4 + k],
                                wx[8 + i] * wy[j] * wz[k],     wx[4 + i] * wy[4 + j] * wz[k],
                                wx[4 + i] * wy[j] * wz[4 + k], wx[i] * wy[8 + j] * wz[k],
                                wx[i] * wy[4 + j] * wz[4 + k], wx[i] * wy[j] * wz[8 + k]};
                            for (int s = 0; s < 10; ++s) {
                                double *a = A + (size_t)s * N;
                                double w = pre[s];
                                for (int n = 0; n < N; ++n) a[n] += w * p[n];
                            }
                            if (scale) {
                                for (int s = 0; s < 10; ++s) {
                                    double *b = B + (size_t)s * N;
                                    double w = fabs(pre[s]);
                                    for (int n = 0; n < N; ++n) b[n] += w * fabs(p[n]);
                                }
                            }
                        }
                    }
                }
                /* select / combine streams in reference order (oracle.py:105-115) */
                static const int sel_v[1] = {0};
                static const int sel_vgl[4] = {0, 1, 2, 3};
                static const int sel_vgh[10] = {0, 1, 2, 3, 4, 5, 6, 7, 8, 9};
                const int *sel = kind == ORC_V ? sel_v : (kind == ORC_VGL ? sel_vgl : sel_vgh);
                int nsel = kind == ORC_V ? 1 : (kind == ORC_VGL ? 4 : 10);
                double *o = out + q * pos_stride;
                double *sc = scale ? scale + q * pos_stride : NULL;
                for (int s = 0; s < nsel; ++s) {
                    memcpy(o + s * stream_stride, A + (size_t)sel[s] * N, sizeof(double) * (size_t)N);
                    if (sc) memcpy(sc + s * stream_stride, B + (size_t)sel[s] * N, sizeof(double) * (size_t)N);
                }
                if (kind == ORC_VGL) {
                    double *l = o + 4 * stream_stride;
                    for (int n = 0; n < N; ++n)
                        l[n] = A[4 * (size_t)N + n] + A[7 * (size_t)N + n] + A[9 * (size_t)N + n];
                    if (sc) {
                        double *ls = sc + 4 * stream_stride;
                        for (int n = 0; n < N; ++n)
                            ls[n] = B[4 * (size_t)N + n] + B[7 * (size_t)N + n] + B[9 * (size_t)N + n];
                    }
                }
            }
        }
        free(acc);
        free(p);
    }
    return err;
}

int orc_abi_version(void) { return 1; }

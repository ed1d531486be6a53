// spo_eval.cu -- fused V / VGL / VGH gather-contract kernels for sm_100a.
//
// Reference: kernels.py:132-247 (_prep + _v_soa/_vgl_soa/_vgh_soa) and the
// batch drivers kernels.py:357-381; dispatch kernels.py:445-473.
//
// One CTA = (a block of `ppc` positions) x (one orbital chunk of one tile).
// Grid: x = position block (fastest) -> all position blocks of chunk 0 run
// before chunk 1 (tile-major, the paper's AoSoA cache blocking: one tile
// slice of the table is the L2 working set at a time).  Threads: blockDim.x =
// `chv` 16-byte orbital vectors (float4 / double2) along the row, blockDim.y =
// position groups; each group walks its positions.
//
// Prologue (fused): the first `ppc` threads map their position to (i0,j0,k0)
// and 36 basis weights bit-exactly (spo_prologue.cuh) into shared memory.
//
// Contraction, per position and 16-byte lane vector:
//   FAST   separable: s_b = sum_k wz_b[k] c[k]   (b = 0,1,2 derivative order)
//                     t_ab += wy_a[j] s_b         (per i, 6 combos for VGH)
//                     acc  += wx_c[i] t_ab        (10 streams)
//          = 328 FMA / orbital for VGH (vs 640 mul+add in the reference).
//   STRICT the reference order i, j, k with fp32 prefactors (a_i*a_j)*a_k and
//          acc = acc + pre*c as separate round-to-nearest mul and add -- bitwise
//          equal to the numba kernels (kernels.py:219-247, 189 for `pl`).
// Loads are 16-byte read-only (ld.global.nc) row reads, coalesced across the
// warp; stores are 16-byte streaming (st.global.cs) so outputs do not evict
// the table from L2.
#include "spo_common.cuh"
#include "spo_prologue.cuh"

#include <cstdlib>

namespace spo {

template <typename T>
struct Vec;
template <>
struct Vec<float> {
    static constexpr int W = 4;
};
template <>
struct Vec<double> {
    static constexpr int W = 2;
};

__device__ __forceinline__ void ld16(const float *p, float *r) {
    float4 v = __ldg(reinterpret_cast<const float4 *>(p));
    r[0] = v.x;
    r[1] = v.y;
    r[2] = v.z;
    r[3] = v.w;
}
__device__ __forceinline__ void ld16(const double *p, double *r) {
    double2 v = __ldg(reinterpret_cast<const double2 *>(p));
    r[0] = v.x;
    r[1] = v.y;
}
__device__ __forceinline__ void st16(float *p, const float *r) {
    __stcs(reinterpret_cast<float4 *>(p), make_float4(r[0], r[1], r[2], r[3]));
}
__device__ __forceinline__ void st16(double *p, const double *r) {
    __stcs(reinterpret_cast<double2 *>(p), make_double2(r[0], r[1]));
}
__device__ __forceinline__ float fmaT(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fmaT(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float addT(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double addT(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float mulT(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mulT(double a, double b) { return __dmul_rn(a, b); }

template <int KIND>
struct Streams {
    static constexpr int S = KIND == SPO_KIND_V ? 1 : (KIND == SPO_KIND_VGL ? 5 : 10);
};

struct EvalArgs {
    const void *table;
    long long tile_stride;
    int nb;
    int chv;              // 16-byte vectors per chunk (= blockDim.x)
    int chunks_per_tile;  // nb / (chv * W)
    long long si, sj, sk; // element strides of i', j', k'
    int nyp, nzp;
    const double *pos;
    long long n_pos;
    int ppc;              // positions per CTA
    GridArgs g;
    void *out;
    long long out_pos_stride, out_stream_stride;
    const long long *out_index;
    long long lane_limit;  // output lanes >= lane_limit are not stored
    int *status;
    int kmul;              // k-power tables: cell k0's rows start at 4 k0
    double dz, dz2;        // k-power tables: 1/dz, 2/dz^2
};

// ---------------------------------------------------------------- FAST ----
//   KP     k-power tables (spo_b200.h SPO_TABLE_KPOWER): the four rows are the
//          power-basis q0..q3 of the z-cubic; A, D, H as spo_tma.cuh kpow_sums
//          (w[24] = t_z), 1/dz and 2/dz^2 folded into the x weights -- the
//          sequence of the TMA and line kernels' slab_contract_kp (bitwise).
template <int KIND, typename T, bool KP>
__device__ __forceinline__ void contract_fast(const T *__restrict__ rp, long long si, long long sj,
                                              long long sk, const T *__restrict__ w, T dz, T dz2,
                                              T (&acc)[Streams<KIND>::S][Vec<T>::W]) {
    constexpr int W = Vec<T>::W;
    T wx[12], wy[12], wz[12];
#pragma unroll
    for (int e = 0; e < 12; ++e) {
        wx[e] = w[e];
        wy[e] = w[12 + e];
        wz[e] = w[24 + e];
    }
#pragma unroll
    for (int s = 0; s < Streams<KIND>::S; ++s)
#pragma unroll
        for (int e = 0; e < W; ++e) acc[s][e] = T(0);
    // fp32 B-spline tables: the z second derivative through the (ax ay)-weighted
    // z rows, as spo_tma.cuh slab_contract / finish_z2 (same sequence, bitwise)
    constexpr bool Z2 = !KP && sizeof(T) == 4 && KIND != SPO_KIND_V;
    T zs[4][W];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int e = 0; e < W; ++e) zs[c][e] = T(0);

#pragma unroll
    for (int i = 0; i < 4; ++i) {
        // t_ab: y-derivative order a, z-derivative order b
        T t00[W], t10[W], t01[W], t20[W], t11[W], t02[W];
#pragma unroll
        for (int e = 0; e < W; ++e) t00[e] = t10[e] = t01[e] = t20[e] = t11[e] = t02[e] = T(0);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const T *r = rp + i * si + j * sj;
            T c0[W], c1[W], c2[W], c3[W];
            ld16(r, c0);
            ld16(r + sk, c1);
            ld16(r + 2 * sk, c2);
            ld16(r + 3 * sk, c3);
            const T axy = mulT(wx[i], wy[j]);
#pragma unroll
            for (int e = 0; e < W; ++e) {
                T s0, s1, s2;
                if constexpr (KP) {
                    const T tz = wz[0];
                    const T q = fmaT(tz, c3[e], c2[e]);  // q2 + t q3
                    s0 = fmaT(tz, fmaT(tz, q, c1[e]), c0[e]);
                    if (KIND != SPO_KIND_V) {
                        const T h = fmaT(tz, c3[e], q);  // q2 + 2t q3
                        s1 = fmaT(tz, addT(q, h), c1[e]);
                        s2 = fmaT(tz, c3[e], h);
                    }
                } else {
                    s0 = fmaT(wz[3], c3[e], fmaT(wz[2], c2[e], fmaT(wz[1], c1[e], wz[0] * c0[e])));
                    if (KIND != SPO_KIND_V) {
                        s1 = fmaT(wz[7], c3[e], fmaT(wz[6], c2[e], fmaT(wz[5], c1[e], wz[4] * c0[e])));
                        if constexpr (!Z2)
                            s2 = fmaT(wz[11], c3[e], fmaT(wz[10], c2[e], fmaT(wz[9], c1[e], wz[8] * c0[e])));
                    }
                }
                t00[e] = fmaT(wy[j], s0, t00[e]);
                if (KIND != SPO_KIND_V) {
                    t10[e] = fmaT(wy[4 + j], s0, t10[e]);
                    t01[e] = fmaT(wy[j], s1, t01[e]);
                    t20[e] = fmaT(wy[8 + j], s0, t20[e]);
                    if (KIND == SPO_KIND_VGH) t11[e] = fmaT(wy[4 + j], s1, t11[e]);
                    if constexpr (Z2) {
                        zs[0][e] = fmaT(axy, c0[e], zs[0][e]);
                        zs[1][e] = fmaT(axy, c1[e], zs[1][e]);
                        zs[2][e] = fmaT(axy, c2[e], zs[2][e]);
                        zs[3][e] = fmaT(axy, c3[e], zs[3][e]);
                    } else {
                        t02[e] = fmaT(wy[j], s2, t02[e]);
                    }
                }
            }
        }
        // z-derivative x weights: the B-spline form carries 1/dz in wz; the
        // k-power form folds it here (axz = ax/dz, daxz = dax/dz, axz2 = 2ax/dz^2)
        const T axz = KP ? mulT(wx[i], dz) : wx[i], daxz = KP ? mulT(wx[4 + i], dz) : wx[4 + i];
        const T axz2 = KP ? mulT(wx[i], dz2) : wx[i];
#pragma unroll
        for (int e = 0; e < W; ++e) {
            acc[0][e] = fmaT(wx[i], t00[e], acc[0][e]);
            if (KIND != SPO_KIND_V) {
                acc[1][e] = fmaT(wx[4 + i], t00[e], acc[1][e]);  // gx
                acc[2][e] = fmaT(wx[i], t10[e], acc[2][e]);      // gy
                acc[3][e] = fmaT(axz, t01[e], acc[3][e]);        // gz
            }
            if (KIND == SPO_KIND_VGL) {
                // l = d2x*t00 + x*t20 + x*t02 (Z2: the z term after the loop)
                if constexpr (Z2)
                    acc[4][e] = fmaT(wx[8 + i], t00[e], fmaT(wx[i], t20[e], acc[4][e]));
                else
                    acc[4][e] = fmaT(wx[8 + i], t00[e], fmaT(wx[i], t20[e], fmaT(axz2, t02[e], acc[4][e])));
            }
            if (KIND == SPO_KIND_VGH) {
                acc[4][e] = fmaT(wx[8 + i], t00[e], acc[4][e]);  // hxx
                acc[5][e] = fmaT(wx[4 + i], t10[e], acc[5][e]);  // hxy
                acc[6][e] = fmaT(daxz, t01[e], acc[6][e]);       // hxz
                acc[7][e] = fmaT(wx[i], t20[e], acc[7][e]);      // hyy
                acc[8][e] = fmaT(axz, t11[e], acc[8][e]);        // hyz
                if constexpr (!Z2) acc[9][e] = fmaT(axz2, t02[e], acc[9][e]);  // hzz
            }
        }
    }
    if constexpr (Z2) {
#pragma unroll
        for (int e = 0; e < W; ++e) {
            const T zz = fmaT(wz[11], zs[3][e], fmaT(wz[10], zs[2][e], fmaT(wz[9], zs[1][e], wz[8] * zs[0][e])));
            if (KIND == SPO_KIND_VGH) acc[9][e] = zz;
            if (KIND == SPO_KIND_VGL) acc[4][e] = addT(acc[4][e], zz);
        }
    }
}

// -------------------------------------------------------------- STRICT ----
// kernels.py:219-247 (VGH), 178-196 (VGL), 152-161 (V): fp32, no FMA.
template <int KIND>
__device__ __forceinline__ void contract_strict(const float *__restrict__ rp, long long si,
                                                long long sj, long long sk,
                                                const float *__restrict__ w,
                                                float (&acc)[Streams<KIND>::S][4]) {
    float wx[12], wy[12], wz[12];
#pragma unroll
    for (int e = 0; e < 12; ++e) {
        wx[e] = w[e];
        wy[e] = w[12 + e];
        wz[e] = w[24 + e];
    }
#pragma unroll
    for (int s = 0; s < Streams<KIND>::S; ++s)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[s][e] = 0.0f;
#define MUL3(a, b, c) __fmul_rn(__fmul_rn((a), (b)), (c))
#pragma unroll
    for (int i = 0; i < 4; ++i) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                float c[4];
                ld16(rp + i * si + j * sj + k * sk, c);
                const float ax = wx[i], dax = wx[4 + i], d2ax = wx[8 + i];
                const float ay = wy[j], day = wy[4 + j], d2ay = wy[8 + j];
                const float az = wz[k], daz = wz[4 + k], d2az = wz[8 + k];
                float pre[Streams<KIND>::S];
                pre[0] = MUL3(ax, ay, az);
                if (KIND != SPO_KIND_V) {
                    pre[1] = MUL3(dax, ay, az);
                    pre[2] = MUL3(ax, day, az);
                    pre[3] = MUL3(ax, ay, daz);
                }
                if (KIND == SPO_KIND_VGL) {
                    // kernels.py:189: d2ax*ay*az + ax*d2ay*az + ax*ay*d2az
                    pre[4] = __fadd_rn(__fadd_rn(MUL3(d2ax, ay, az), MUL3(ax, d2ay, az)),
                                       MUL3(ax, ay, d2az));
                }
                if (KIND == SPO_KIND_VGH) {
                    pre[4] = MUL3(d2ax, ay, az);
                    pre[5] = MUL3(dax, day, az);
                    pre[6] = MUL3(dax, ay, daz);
                    pre[7] = MUL3(ax, d2ay, az);
                    pre[8] = MUL3(ax, day, daz);
                    pre[9] = MUL3(ax, ay, d2az);
                }
#pragma unroll
                for (int s = 0; s < Streams<KIND>::S; ++s)
#pragma unroll
                    for (int e = 0; e < 4; ++e) acc[s][e] = __fadd_rn(acc[s][e], __fmul_rn(pre[s], c[e]));
            }
        }
    }
#undef MUL3
}

// -------------------------------------------------------------- kernel ----
template <int KIND, typename T, bool STRICT, bool KP>
__global__ void __launch_bounds__(256, 1) eval_kernel(const EvalArgs a) {
    constexpr int W = Vec<T>::W;
    constexpr int S = Streams<KIND>::S;
    extern __shared__ __align__(16) unsigned char smem[];
    T *sw = reinterpret_cast<T *>(smem);                                  // [ppc][36]
    long long *sbase = reinterpret_cast<long long *>(sw + a.ppc * 36);    // [ppc]

    const int nthr = blockDim.x * blockDim.y;
    const int tid = threadIdx.y * blockDim.x + threadIdx.x;
    const long long p0 = (long long)blockIdx.x * a.ppc;
    const int np = (int)min((long long)a.ppc, a.n_pos - p0);

    for (int q = tid; q < np; q += nthr) {
        const double *r = a.pos + 3 * (p0 + q);
        const double x = r[0], y = r[1], z = r[2];
        double tx, ty, tz;
        const int i0 = map_axis(x, a.g.dinv[0], a.g.cnt[0], &tx);
        const int j0 = map_axis(y, a.g.dinv[1], a.g.cnt[1], &ty);
        const int k0 = map_axis(z, a.g.dinv[2], a.g.cnt[2], &tz);
        axis_weights<T>(tx, a.g.dinv[0], a.g.delta[0], sw + q * 36);
        axis_weights<T>(ty, a.g.dinv[1], a.g.delta[1], sw + q * 36 + 12);
        axis_weights<T>(tz, a.g.dinv[2], a.g.delta[2], sw + q * 36 + 24);
        if (KP) sw[q * 36 + 24] = (T)tz;
        const bool finite = isfinite(x) && isfinite(y) && isfinite(z);
        sbase[q] = finite ? ((long long)i0 * a.nyp + j0) * a.nzp * a.nb + (long long)k0 * a.kmul * a.nb : -1;
        if (!finite && a.status) atomicOr(a.status, 1);
    }
    __syncthreads();

    const int m = blockIdx.y / a.chunks_per_tile;
    const int c = blockIdx.y - m * a.chunks_per_tile;
    const int vlane = c * a.chv + threadIdx.x;
    const T *tb = reinterpret_cast<const T *>(a.table) + (long long)m * a.tile_stride + (long long)vlane * W;
    const long long lane0 = (long long)m * a.nb + (long long)vlane * W;

    for (int q = threadIdx.y; q < np; q += blockDim.y) {
        const long long base = sbase[q];
        T acc[S][W];
        if (base >= 0) {
            if constexpr (STRICT) {
                contract_strict<KIND>(tb + base, a.si, a.sj, a.sk, sw + q * 36, acc);
            } else {
                contract_fast<KIND, T, KP>(tb + base, a.si, a.sj, a.sk, sw + q * 36, (T)a.dz, (T)a.dz2, acc);
            }
        } else {
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
                for (int e = 0; e < W; ++e) acc[s][e] = T(NAN);
        }
        const long long op = a.out_index ? a.out_index[p0 + q] : p0 + q;
        T *o = reinterpret_cast<T *>(a.out) + op * a.out_pos_stride + lane0;
        if (lane0 + W <= a.lane_limit) {
#pragma unroll
            for (int s = 0; s < S; ++s) st16(o + s * a.out_stream_stride, acc[s]);
        } else if (lane0 < a.lane_limit) {  // the vector straddles lane_limit
            const int nv = (int)(a.lane_limit - lane0);
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
                for (int e = 0; e < W - 1; ++e)
                    if (e < nv) o[s * a.out_stream_stride + e] = acc[s][e];
        }
    }
}

template <int KIND, typename T, bool STRICT, bool KP = false>
static int launch(const EvalArgs &a, dim3 grid, dim3 block, size_t smem, cudaStream_t st) {
    eval_kernel<KIND, T, STRICT, KP><<<grid, block, smem, st>>>(a);
    return check_launch("spo_eval launch");
}

}  // namespace spo

namespace spo {
int eval_tma(int kind, int dtype, const void *table, const TableGeom &geo, const GridArgs &g, const double *pos,
             long long n_pos, void *out, long long ops, long long oss, const long long *out_index, int *status,
             void *workspace, long long ws_bytes, cudaStream_t st, int cw_request, long long lane_limit,
             const void *coef = nullptr, long long coef_stride = 0, double *ratios = nullptr);
long long eval_tma_workspace_bytes(int dtype, long long n_pos);
long long eval_line_workspace_bytes(int dtype, long long n_pos);
bool eval_line_eligible(int dtype, const TableGeom &geo, long long n_pos, long long ws_bytes);
int eval_line(int kind, int dtype, const void *table, const TableGeom &geo, const GridArgs &g, const double *pos,
              long long n_pos, void *out, long long ops, long long oss, const long long *out_index, int *status,
              void *workspace, long long ws_bytes, cudaStream_t st, long long lane_limit,
              const void *coef = nullptr, long long coef_stride = 0, double *ratios = nullptr,
              long long ratio_bytes = 0, int win = 1);
int line_window_cells();
int line_v_window();
long long eval_tma_ratio_bytes(int kind, int dtype, long long nb, long long n_tiles, long long n_pos);
}

using namespace spo;

extern "C" int spo_abi_version(void) { return SPO_ABI_VERSION; }

extern "C" const char *spo_last_error(void) { return last_error_slot().c_str(); }

extern "C" int64_t spo_eval_workspace_bytes(int kind, int dtype, int mode, int64_t n_pos) {
    if (kind < SPO_KIND_V || kind > SPO_KIND_VGH || n_pos < 0) return -1;
    mode &= ~SPO_TABLE_KPOWER;
    if ((dtype != SPO_F32 && dtype != SPO_F64) || mode != SPO_MODE_FAST) return 0;
    const long long a = eval_tma_workspace_bytes(dtype, n_pos), b = eval_line_workspace_bytes(dtype, n_pos);
    return a > b ? a : b;
}

// Shared-plane kernels by density (positions per grid cell; sustained
// interleaved timings, scripts/micro/window_ab.py, profiles/r02/window_ab.md):
// the per-position TMA kernel below WINDOW_MIN_*; the window variant of the
// line kernel ((2+3) x (2+3)-row planes shared by the positions of 2 x 2
// (j0, k0) cells: +4% at 0.3/cell, +15-20% at 0.5-1/cell over the
// per-position kernel, +1-5% over the line kernel up to 2.4/cell); the line
// kernel from LINE_MIN_* (many positions per line: its V position groups
// and fewer plane loads per slot pay).  V from VWIN_MIN_V* per cell to the
// line kernel: the 2 x 1 window (planes of two lines along j) with V
// position groups, 7-16% ahead of both the 2 x 2 window and the line kernel
// there (profiles/r02/v_window.md; thresholds re-measured with the dynamic V
// groups, profiles/r02/v_dynamic.md: fp32 2 x 1 window from 1.1, line from
// 2.8; fp64 2 x 1 window from 1.3, line from 4).  k-power tables: no window variant (rows
// have no z halo), the line kernel from 1 (VGL/VGH) / 2 (V) per cell.
constexpr double WINDOW_MIN_VGX = 0.3, WINDOW_MIN_V = 0.4, VWIN_MIN_V32 = 1.1, VWIN_MIN_V64 = 1.3;
constexpr double LINE_MIN_VGX = 4.0, LINE_MIN_V32 = 2.8, LINE_MIN_V64 = 4.0;
constexpr double KP_LINE_MIN_VGX = 1.0, KP_LINE_MIN_V = 2.0;

// Which shared-plane kernel a FAST request takes: 0 = none (the per-position
// TMA kernel), 1 = the line kernel, 3 = its 2 x 2 window variant, 4 = the
// 2 x 1 window with V position groups (V only).  SPO_LINE=0/1/2 forces none
// / line / a window (read on every call; SPO_VWIN=0/1 then picks which for V).
static int line_variant(int kind, int dtype, const int32_t *n3, long long n_pos, bool kpower) {
    const double dens = (double)n_pos / ((double)n3[0] * n3[1] * n3[2]);
    const bool v = kind == SPO_KIND_V;
    auto window = [&]() {
        const char *e = getenv("SPO_VWIN");
        const bool vw = v && (e ? e[0] == '1' : dens >= (dtype == SPO_F64 ? VWIN_MIN_V64 : VWIN_MIN_V32));
        return vw ? 4 : 3;
    };
    const char *env_line = getenv("SPO_LINE");
    if (env_line) return env_line[0] == '1' ? 1 : (env_line[0] == '2' && !kpower ? window() : 0);
    if (kpower) return dens >= (v ? KP_LINE_MIN_V : KP_LINE_MIN_VGX) ? 1 : 0;
    if (dens >= (v ? (dtype == SPO_F64 ? LINE_MIN_V64 : LINE_MIN_V32) : LINE_MIN_VGX)) return 1;
    return dens >= (v ? WINDOW_MIN_V : WINDOW_MIN_VGX) ? window() : 0;
}

// lane_limit < 0: every table lane is stored and `out` must be memory of the
// launch device (bound from `out`).  lane_limit >= 0 (spo_eval_lanes): lanes
// [0, lane_limit) are stored, the launch device is the table's and `out` may
// be peer memory reachable from it.
static int eval_impl(int kind, int dtype, int mode, const void *table, const int32_t *n3, int32_t nb,
                     int32_t n_tiles, const double *dinv3, const double *delta3, const double *pos, int64_t n_pos,
                     void *out, int64_t out_pos_stride, int64_t out_stream_stride, int64_t lane_limit,
                     const int64_t *out_index, int32_t *status, void *workspace, int64_t workspace_bytes,
                     void *stream) {
    if (kind < SPO_KIND_V || kind > SPO_KIND_VGH) return fail(SPO_ERR_CONTRACT, "unknown kind %d", kind);
    if (dtype != SPO_F32 && dtype != SPO_F64) return fail(SPO_ERR_CONTRACT, "unknown dtype %d", dtype);
    const bool kpower = (mode & SPO_TABLE_KPOWER) != 0;
    mode &= ~SPO_TABLE_KPOWER;
    if (mode != SPO_MODE_FAST && mode != SPO_MODE_STRICT) return fail(SPO_ERR_CONTRACT, "unknown mode %d", mode);
    if (mode == SPO_MODE_STRICT && dtype != SPO_F32)
        return fail(SPO_ERR_CONFIG, "strict mode reproduces the fp32 reference kernels only");
    if (mode == SPO_MODE_STRICT && kpower)
        return fail(SPO_ERR_CONFIG, "strict mode needs the B-spline table form (the reference's arithmetic)");
    TableGeom geo;
    int rc = make_geom(n3, nb, n_tiles, dtype, &geo, kpower);
    if (rc) return rc;
    if (n_pos < 0) return fail(SPO_ERR_CONTRACT, "n_pos=%lld < 0", (long long)n_pos);
    if (n_pos == 0) return ok();
    if (!table || !pos || !out || !dinv3 || !delta3) return fail(SPO_ERR_CONTRACT, "NULL pointer argument");
    const int W = dtype == SPO_F64 ? 2 : 4;
    const int S = kind == SPO_KIND_V ? 1 : (kind == SPO_KIND_VGL ? 5 : 10);
    if (!aligned16(table) || !aligned16(out))
        return fail(SPO_ERR_CONTRACT, "table and out must be 16-byte aligned");
    if (out_pos_stride % W || out_stream_stride % W)
        return fail(SPO_ERR_CONTRACT, "output strides must be multiples of %d elements", W);
    const bool peer = lane_limit >= 0;
    const long long table_lanes = (long long)nb * n_tiles;
    if (peer && (lane_limit == 0 || lane_limit > table_lanes))
        return fail(SPO_ERR_CONTRACT, "lane_limit %lld outside [1, %lld]", (long long)lane_limit, table_lanes);
    const long long lanes = peer ? (long long)lane_limit : table_lanes;
    if (S > 1 && out_stream_stride < lanes)
        return fail(SPO_ERR_CONTRACT, "out_stream_stride %lld shorter than the %lld table lanes",
                    (long long)out_stream_stride, lanes);
    if (out_pos_stride < (long long)(S - 1) * out_stream_stride + lanes && !(n_pos == 1 && !out_index))
        return fail(SPO_ERR_CONTRACT, "out_pos_stride %lld too small for %d streams",
                    (long long)out_pos_stride, S);
    for (int ax = 0; ax < 3; ++ax)
        if (!(dinv3[ax] > 0.0) || !(delta3[ax] > 0.0))
            return fail(SPO_ERR_CONFIG, "grid spacing on axis %d must be positive", ax);

    rc = peer ? bind_device(table) : bind_device(out);
    if (rc) return rc;
    if ((rc = check_on_device(table, "table")) || (rc = check_on_device(pos, "positions")) ||
        (rc = check_on_device(out_index, "out_index")) || (rc = check_on_device(status, "status")) ||
        (rc = check_on_device(workspace, "workspace")) ||
        (rc = peer ? check_reachable(out, "out") : SPO_OK))
        return rc;
    if (mode == SPO_MODE_FAST) {
        static const char *env_tma = getenv("SPO_TMA");
        static const char *env_cw = getenv("SPO_CW");
        if (!(env_tma && env_tma[0] == '0')) {
            GridArgs g;
            for (int ax = 0; ax < 3; ++ax) {
                g.dinv[ax] = dinv3[ax];
                g.cnt[ax] = (double)n3[ax];
                g.delta[ax] = delta3[ax];
                g.n[ax] = n3[ax];
            }
            const int lv = line_variant(kind, dtype, n3, n_pos, kpower);
            if (lv) {
                const int r = eval_line(kind, dtype, table, geo, g, pos, n_pos, out, out_pos_stride,
                                        out_stream_stride, reinterpret_cast<const long long *>(out_index), status,
                                        workspace, workspace_bytes, reinterpret_cast<cudaStream_t>(stream), lanes,
                                        nullptr, 0, nullptr, 0,
                                        lv == 4 ? line_v_window() : (lv == 3 ? line_window_cells() : 1));
                if (r >= 0) return r;
            }
            const int r = eval_tma(kind, dtype, table, geo, g, pos, n_pos, out, out_pos_stride, out_stream_stride,
                                   reinterpret_cast<const long long *>(out_index), status, workspace,
                                   workspace_bytes, reinterpret_cast<cudaStream_t>(stream),
                                   env_cw ? atoi(env_cw) : 0, lanes);
            if (r >= 0) return r;
        }
    }

    EvalArgs a;
    a.table = table;
    a.tile_stride = geo.tile_stride;
    a.nb = nb;
    const int Q = nb / W;  // 16-byte vectors per row, multiple of 8
    int chv = 8;
    for (int d = 8; d <= 256 && d <= Q; d += 8)
        if (Q % d == 0) chv = d;
    a.chv = chv;
    a.chunks_per_tile = Q / chv;
    a.sk = nb;
    a.sj = (long long)geo.nzp * nb;
    a.si = (long long)geo.nyp * geo.nzp * nb;
    a.nyp = geo.nyp;
    a.nzp = geo.nzp;
    a.pos = pos;
    a.n_pos = n_pos;
    for (int ax = 0; ax < 3; ++ax) {
        a.g.dinv[ax] = dinv3[ax];
        a.g.cnt[ax] = (double)n3[ax];
        a.g.delta[ax] = delta3[ax];
        a.g.n[ax] = n3[ax];
    }
    a.out = out;
    a.out_pos_stride = out_pos_stride;
    a.out_stream_stride = out_stream_stride;
    a.out_index = reinterpret_cast<const long long *>(out_index);
    a.lane_limit = lanes;
    a.status = status;
    a.kmul = geo.kmul;
    a.dz = dinv3[2];
    a.dz2 = 2.0 * dinv3[2] * dinv3[2];

    const int groups = 256 / chv;
    const long long n_chunks = (long long)a.chunks_per_tile * n_tiles;
    if (n_chunks > 65535) return fail(SPO_ERR_CONFIG, "too many orbital chunks (%lld)", n_chunks);
    // positions per CTA: up to 4 per group while keeping >= 4 CTAs per SM
    int ppg = 4;
    while (ppg > 1 && ((n_pos + (long long)groups * ppg - 1) / ((long long)groups * ppg)) * n_chunks < 4 * 148)
        ppg >>= 1;
    a.ppc = groups * ppg;
    const long long nblk = (n_pos + a.ppc - 1) / a.ppc;
    if (nblk > 0x7fffffffLL) return fail(SPO_ERR_CONFIG, "too many positions");
    dim3 grid((unsigned)nblk, (unsigned)n_chunks);
    dim3 block(chv, groups);
    const size_t smem = (size_t)a.ppc * (36 * (size_t)(dtype == SPO_F64 ? 8 : 4) + 8);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);

    if (kpower) {
        if (dtype == SPO_F64) {
            switch (kind) {
                case SPO_KIND_V: return launch<SPO_KIND_V, double, false, true>(a, grid, block, smem, st);
                case SPO_KIND_VGL: return launch<SPO_KIND_VGL, double, false, true>(a, grid, block, smem, st);
                default: return launch<SPO_KIND_VGH, double, false, true>(a, grid, block, smem, st);
            }
        }
        switch (kind) {
            case SPO_KIND_V: return launch<SPO_KIND_V, float, false, true>(a, grid, block, smem, st);
            case SPO_KIND_VGL: return launch<SPO_KIND_VGL, float, false, true>(a, grid, block, smem, st);
            default: return launch<SPO_KIND_VGH, float, false, true>(a, grid, block, smem, st);
        }
    }
    if (dtype == SPO_F64) {
        switch (kind) {
            case SPO_KIND_V: return launch<SPO_KIND_V, double, false>(a, grid, block, smem, st);
            case SPO_KIND_VGL: return launch<SPO_KIND_VGL, double, false>(a, grid, block, smem, st);
            default: return launch<SPO_KIND_VGH, double, false>(a, grid, block, smem, st);
        }
    }
    if (mode == SPO_MODE_STRICT) {
        switch (kind) {
            case SPO_KIND_V: return launch<SPO_KIND_V, float, true>(a, grid, block, smem, st);
            case SPO_KIND_VGL: return launch<SPO_KIND_VGL, float, true>(a, grid, block, smem, st);
            default: return launch<SPO_KIND_VGH, float, true>(a, grid, block, smem, st);
        }
    }
    switch (kind) {
        case SPO_KIND_V: return launch<SPO_KIND_V, float, false>(a, grid, block, smem, st);
        case SPO_KIND_VGL: return launch<SPO_KIND_VGL, float, false>(a, grid, block, smem, st);
        default: return launch<SPO_KIND_VGH, float, false>(a, grid, block, smem, st);
    }
}

extern "C" int spo_eval_path(int kind, int dtype, int mode, const int32_t *n3, int32_t nb, int32_t n_tiles,
                             int64_t n_pos, int64_t workspace_bytes) {
    if (kind < SPO_KIND_V || kind > SPO_KIND_VGH || (dtype != SPO_F32 && dtype != SPO_F64) || n_pos < 0) return -1;
    const bool kpower = (mode & SPO_TABLE_KPOWER) != 0;
    mode &= ~SPO_TABLE_KPOWER;
    if (kpower && mode != SPO_MODE_FAST) return -1;
    TableGeom geo;
    if (make_geom(n3, nb, n_tiles, dtype, &geo, kpower)) return -1;
    if (mode != SPO_MODE_FAST || workspace_bytes <= 0) return SPO_PATH_GENERIC;
    const char *env_tma = getenv("SPO_TMA");
    if (env_tma && env_tma[0] == '0') return SPO_PATH_GENERIC;
    const int lv = line_variant(kind, dtype, n3, n_pos, kpower);
    if (lv && eval_line_eligible(dtype, geo, n_pos, workspace_bytes)) return lv >= 3 ? SPO_PATH_WINDOW : SPO_PATH_LINE;
    if (workspace_bytes >= eval_tma_workspace_bytes(dtype, n_pos) && n_pos < (1LL << 31)) return SPO_PATH_TMA;
    return SPO_PATH_GENERIC;
}

extern "C" int spo_eval(int kind, int dtype, int mode, const void *table, const int32_t *n3,
                        int32_t nb, int32_t n_tiles, const double *dinv3, const double *delta3,
                        const double *pos, int64_t n_pos, void *out, int64_t out_pos_stride,
                        int64_t out_stream_stride, const int64_t *out_index, int32_t *status,
                        void *workspace, int64_t workspace_bytes, void *stream) {
    return eval_impl(kind, dtype, mode, table, n3, nb, n_tiles, dinv3, delta3, pos, n_pos, out, out_pos_stride,
                     out_stream_stride, -1, out_index, status, workspace, workspace_bytes, stream);
}

extern "C" int spo_eval_lanes(int kind, int dtype, int mode, const void *table, const int32_t *n3,
                              int32_t nb, int32_t n_tiles, const double *dinv3, const double *delta3,
                              const double *pos, int64_t n_pos, void *out, int64_t out_pos_stride,
                              int64_t out_stream_stride, int64_t lane_limit, const int64_t *out_index,
                              int32_t *status, void *workspace, int64_t workspace_bytes, void *stream) {
    if (lane_limit < 0) return fail(SPO_ERR_CONTRACT, "lane_limit %lld < 0", (long long)lane_limit);
    return eval_impl(kind, dtype, mode, table, n3, nb, n_tiles, dinv3, delta3, pos, n_pos, out, out_pos_stride,
                     out_stream_stride, lane_limit, out_index, status, workspace, workspace_bytes, stream);
}

// ------------------------------------------------------------ ratios ----
extern "C" int64_t spo_eval_ratios_workspace_bytes(int kind, int dtype, int32_t nb, int32_t n_tiles,
                                                   int64_t n_pos) {
    if (kind < SPO_KIND_V || kind > SPO_KIND_VGH || n_pos < 0 || nb <= 0 || n_tiles <= 0) return -1;
    if (dtype != SPO_F32 && dtype != SPO_F64) return -1;
    const long long extra = eval_tma_ratio_bytes(kind, dtype, nb, n_tiles, n_pos);
    if (extra < 0) return -1;
    const long long a = eval_tma_workspace_bytes(dtype, n_pos), b = eval_line_workspace_bytes(dtype, n_pos);
    return (a > b ? a : b) + extra;
}

extern "C" int spo_eval_ratios(int kind, int dtype, const void *table, const int32_t *n3, int32_t nb,
                               int32_t n_tiles, const double *dinv3, const double *delta3, const double *pos,
                               int64_t n_pos, const void *coef, int64_t coef_stride, double *ratios,
                               int32_t *status, void *workspace, int64_t workspace_bytes, void *stream) {
    if (kind < SPO_KIND_V || kind > SPO_KIND_VGH) return fail(SPO_ERR_CONTRACT, "unknown kind %d", kind);
    if (dtype != SPO_F32 && dtype != SPO_F64) return fail(SPO_ERR_CONTRACT, "unknown dtype %d", dtype);
    TableGeom geo;
    int rc = make_geom(n3, nb, n_tiles, dtype, &geo);
    if (rc) return rc;
    if (n_pos < 0) return fail(SPO_ERR_CONTRACT, "n_pos=%lld < 0", (long long)n_pos);
    if (n_pos == 0) return ok();
    if (!table || !pos || !coef || !ratios || !dinv3 || !delta3 || !workspace)
        return fail(SPO_ERR_CONTRACT, "NULL pointer argument");
    const int W = dtype == SPO_F64 ? 2 : 4;
    if (!aligned16(table) || !aligned16(coef) || coef_stride % W)
        return fail(SPO_ERR_CONTRACT, "table/coef must be 16-byte aligned, coef_stride a multiple of %d", W);
    if (coef_stride < (long long)nb * n_tiles)
        return fail(SPO_ERR_CONTRACT, "coef_stride %lld shorter than the %lld table lanes", (long long)coef_stride,
                    (long long)nb * n_tiles);
    for (int ax = 0; ax < 3; ++ax)
        if (!(dinv3[ax] > 0.0) || !(delta3[ax] > 0.0))
            return fail(SPO_ERR_CONFIG, "grid spacing on axis %d must be positive", ax);
    rc = bind_device(ratios);
    if (rc) return rc;
    if ((rc = check_on_device(table, "table")) || (rc = check_on_device(pos, "positions")) ||
        (rc = check_on_device(coef, "coef")) || (rc = check_on_device(status, "status")) ||
        (rc = check_on_device(workspace, "workspace")))
        return rc;
    GridArgs g;
    for (int ax = 0; ax < 3; ++ax) {
        g.dinv[ax] = dinv3[ax];
        g.cnt[ax] = (double)n3[ax];
        g.delta[ax] = delta3[ax];
        g.n[ax] = n3[ax];
    }
    // The line kernel's ratio epilogue only when forced (SPO_LINE=1): without
    // the output stream the per-position kernel is not power-bound, and it is
    // faster (scripts/bench_ratios.py: 6.30e10 vs 6.18e10 orbital-evals/s).
    // V on dense batches is the exception: there the line kernel's position
    // groups (one plane read for 3 positions, aligned to cells) make it 2-3x
    // faster than one position per warp (profiles/r02/rank_share.md), from the
    // densities evaluate() sends V to the line kernel at.  SPO_LINE=0 forces
    // the per-position kernel.
    const char *env_line = getenv("SPO_LINE");
    const double dens = (double)n_pos / ((double)n3[0] * n3[1] * n3[2]);
    const bool dense_v = kind == SPO_KIND_V && dens >= (dtype == SPO_F64 ? 4.0 : 2.8);
    if (env_line ? env_line[0] == '1' : dense_v) {
        const long long extra = eval_tma_ratio_bytes(kind, dtype, nb, n_tiles, n_pos);
        rc = eval_line(kind, dtype, table, geo, g, pos, n_pos, nullptr, 0, 0, nullptr, status, workspace,
                       workspace_bytes, reinterpret_cast<cudaStream_t>(stream), 0, coef, coef_stride, ratios,
                       extra);
        if (rc >= 0) return rc;
    }
    rc = eval_tma(kind, dtype, table, geo, g, pos, n_pos, nullptr, 0, 0, nullptr, status, workspace,
                  workspace_bytes, reinterpret_cast<cudaStream_t>(stream), 0, 0, coef, coef_stride, ratios);
    if (rc < 0) return fail(SPO_ERR_CONFIG, "the fused ratio epilogue is unavailable for this request");
    return rc;
}

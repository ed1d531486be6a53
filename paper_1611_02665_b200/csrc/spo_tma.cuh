// spo_tma.cuh -- TMA / mbarrier / packed-FMA helpers shared by the
// pipelined kernels (spo_eval_tma.cu, spo_eval_line.cu).
#pragma once
#include <cuda.h>

#include "spo_common.cuh"

namespace spo {

// ---- host: the 5-D TMA descriptor of a device table -- dims (lanes, k', j',
// i', tile), box (box_lanes, 4, 4, 1, 1): one box = one (position, i) slab.
// Returns 0, -1 when the driver has no cuTensorMapEncodeTiled, or the
// CUresult of a failed encode.
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn tensor_map_encoder() {
    static const EncodeTiledFn fn = [] {  // thread-safe one-time lookup
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<EncodeTiledFn>(p);
        cudaGetLastError();
        return static_cast<EncodeTiledFn>(nullptr);
    }();
    return fn;
}

// box: box_lanes lanes x box_rows k-rows x box_j j-rows (default box_rows) of
// one i-plane (4 x 4: one position's slab; larger: a window of several
// positions' slabs)
inline int table_tensor_map(CUtensorMap *map, const void *table, const TableGeom &geo, int dtype, int box_lanes,
                            int box_rows = 4, int box_j = 0) {
    if (box_j <= 0) box_j = box_rows;
    EncodeTiledFn encode = tensor_map_encoder();
    if (!encode) return -1;
    const cuuint64_t E = dtype == SPO_F64 ? 8 : 4;
    cuuint64_t dims[5] = {(cuuint64_t)geo.nb, (cuuint64_t)geo.nzp, (cuuint64_t)geo.nyp, (cuuint64_t)geo.nxp,
                          (cuuint64_t)geo.n_tiles};
    cuuint64_t strides[4] = {(cuuint64_t)geo.nb * E, (cuuint64_t)geo.nzp * geo.nb * E,
                             (cuuint64_t)geo.nyp * geo.nzp * geo.nb * E, (cuuint64_t)geo.tile_stride * E};
    cuuint32_t box[5] = {(cuuint32_t)box_lanes, (cuuint32_t)box_rows, (cuuint32_t)box_j, 1, 1};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    const CUresult r =
        encode(map, dtype == SPO_F64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5,
               const_cast<void *>(table), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : (int)r;
}

namespace tma {

__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_test(unsigned long long *bar, unsigned phase) {
    unsigned ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void st_release_shared(unsigned *p, unsigned v) {
    asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned ld_acquire_shared(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}

__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ void tma_load_5d(void *dst, const CUtensorMap *map, unsigned long long *bar, int c0,
                                            int c1, int c2, int c3, int c4, unsigned long long policy) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2], %8;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
        "r"(c4), "l"(policy)
        : "memory");
}

// L2 policy for table slabs: keep the current unit's slice resident while the
// output stream (st.global.cs) passes through.
__device__ __forceinline__ unsigned long long l2_policy(bool evict_last) {
    unsigned long long p;
    if (evict_last)
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    else
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ void bulk_load(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(src)), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int KIND>
struct NS {
    static constexpr int S = KIND == SPO_KIND_V ? 1 : (KIND == SPO_KIND_VGL ? 5 : 10);
};

// ----------------------------------------------------------- contraction --
// Packed fp32x2 FMA (SASS FFMA2, sm_100): two independent round-to-nearest
// fp32 FMAs per instruction with a broadcast scalar multiplier -- bitwise the
// same as two __fmaf_rn, at half the issue slots.
__device__ __forceinline__ float2 fma2(float w, float2 c, float2 acc) {
    return __ffma2_rn(make_float2(w, w), c, acc);
}
__device__ __forceinline__ float2 mul2(float w, float2 c) { return __fmul2_rn(make_float2(w, w), c); }

// One i-slab for one lane: 4 fp32 orbitals as two fp32x2 pairs.
// slab: [j][k][CW] of this lane's position, RJ k-rows per j (4: a slab of its
// own; more: the position's 4 x 4 corner of a window of rows); wy/wz: 12
// weights; ax/dax/d2ax: x weights of this i.
//
// Separable contraction (k, then j, then i), 312 FMAs per orbital for VGH
// (VGL 284).  The z second derivative is the one stream that reaches only
// through (x, y) value weights, so it is not formed per row group like the
// others (4 FMAs on every row group, then a j and an i sum): instead the
// (ax ay)-weighted sums of the four z rows accumulate over the slabs,
// zs[c] += sum_j (ax * ay_j) * c_jc (4 FMAs per row group), and
// finish_z2() contracts them with d2az once per position (4 FMAs).  Every
// product is still (weight) x (coefficient), so the error stays within a
// few ulps of sum|w*c| (the north-star bound).
// The slab contraction in two steps (a kernel that streams a slab row group
// by row group keeps exactly the same arithmetic):
// rowgroup() takes row group j (its 4 k-rows) into the j-sums t, slab_done()
// folds the j-sums into the accumulators with the x weights of this i.
template <int KIND, int J>
__device__ __forceinline__ void rowgroup(const float4 (&c)[4], const float (&wy)[12], const float (&wz)[12],
                                         float ax, float2 (&t)[5][2], float2 (&zs)[4][2]) {
    // t[0..4] = t00, t10, t01, t20, t11
    const float axy = __fmul_rn(ax, wy[J]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const float2 c0 = h ? make_float2(c[0].z, c[0].w) : make_float2(c[0].x, c[0].y);
        const float2 c1 = h ? make_float2(c[1].z, c[1].w) : make_float2(c[1].x, c[1].y);
        const float2 c2 = h ? make_float2(c[2].z, c[2].w) : make_float2(c[2].x, c[2].y);
        const float2 c3 = h ? make_float2(c[3].z, c[3].w) : make_float2(c[3].x, c[3].y);
        const float2 s0 = fma2(wz[3], c3, fma2(wz[2], c2, fma2(wz[1], c1, mul2(wz[0], c0))));
        t[0][h] = fma2(wy[J], s0, t[0][h]);
        if (KIND != SPO_KIND_V) {
            const float2 s1 = fma2(wz[7], c3, fma2(wz[6], c2, fma2(wz[5], c1, mul2(wz[4], c0))));
            t[1][h] = fma2(wy[4 + J], s0, t[1][h]);
            t[2][h] = fma2(wy[J], s1, t[2][h]);
            t[3][h] = fma2(wy[8 + J], s0, t[3][h]);
            if (KIND == SPO_KIND_VGH) t[4][h] = fma2(wy[4 + J], s1, t[4][h]);
            zs[0][h] = fma2(axy, c0, zs[0][h]);
            zs[1][h] = fma2(axy, c1, zs[1][h]);
            zs[2][h] = fma2(axy, c2, zs[2][h]);
            zs[3][h] = fma2(axy, c3, zs[3][h]);
        }
    }
}
template <int KIND>
__device__ __forceinline__ void slab_done(float ax, float dax, float d2ax, const float2 (&t)[5][2],
                                          float2 (&acc)[NS<KIND>::S][2]) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        acc[0][h] = fma2(ax, t[0][h], acc[0][h]);
        if (KIND != SPO_KIND_V) {
            acc[1][h] = fma2(dax, t[0][h], acc[1][h]);
            acc[2][h] = fma2(ax, t[1][h], acc[2][h]);
            acc[3][h] = fma2(ax, t[2][h], acc[3][h]);
        }
        if (KIND == SPO_KIND_VGL) acc[4][h] = fma2(d2ax, t[0][h], fma2(ax, t[3][h], acc[4][h]));  // + zz: finish_z2
        if (KIND == SPO_KIND_VGH) {
            acc[4][h] = fma2(d2ax, t[0][h], acc[4][h]);
            acc[5][h] = fma2(dax, t[1][h], acc[5][h]);
            acc[6][h] = fma2(dax, t[2][h], acc[6][h]);
            acc[7][h] = fma2(ax, t[3][h], acc[7][h]);
            acc[8][h] = fma2(ax, t[4][h], acc[8][h]);
        }
    }
}
template <int KIND, int CW, int RJ = 4>
__device__ __forceinline__ void slab_contract(const float *__restrict__ slab, const float (&wy)[12],
                                              const float (&wz)[12], float ax, float dax, float d2ax,
                                              float2 (&acc)[NS<KIND>::S][2], float2 (&zs)[4][2]) {
    float2 t[5][2];
#pragma unroll
    for (int u = 0; u < 5; ++u) t[u][0] = t[u][1] = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        float4 c[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) c[k] = *reinterpret_cast<const float4 *>(slab + (j * RJ + k) * CW);
        if (j == 0) rowgroup<KIND, 0>(c, wy, wz, ax, t, zs);
        if (j == 1) rowgroup<KIND, 1>(c, wy, wz, ax, t, zs);
        if (j == 2) rowgroup<KIND, 2>(c, wy, wz, ax, t, zs);
        if (j == 3) rowgroup<KIND, 3>(c, wy, wz, ax, t, zs);
    }
    slab_done<KIND>(ax, dax, d2ax, t, acc);
}

// After the four slabs: the z second derivative from the (ax ay)-weighted
// z rows -- VGH: hzz; VGL: added to l (= hxx + hyy + hzz).
template <int KIND>
__device__ __forceinline__ void finish_z2(const float (&wz)[12], const float2 (&zs)[4][2],
                                          float2 (&acc)[NS<KIND>::S][2]) {
    if constexpr (KIND != SPO_KIND_V) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float2 zz = fma2(wz[11], zs[3][h], fma2(wz[10], zs[2][h], fma2(wz[9], zs[1][h], mul2(wz[8], zs[0][h]))));
            if (KIND == SPO_KIND_VGH) acc[9][h] = zz;
            if (KIND == SPO_KIND_VGL) acc[4][h] = __fadd2_rn(acc[4][h], zz);
        }
    }
}

// One i-slab for one lane: 2 fp64 orbitals, DFMA in the generic kernel's
// order; in the same two steps (t[0..5] = t00, t10, t01, t20, t11, t02).
template <int KIND, int J>
__device__ __forceinline__ void rowgroup(const double2 (&c)[4], const double (&wy)[12], const double (&wz)[12],
                                         double (&t)[6][2]) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const double c0 = e ? c[0].y : c[0].x, c1 = e ? c[1].y : c[1].x;
        const double c2 = e ? c[2].y : c[2].x, c3 = e ? c[3].y : c[3].x;
        const double s0 = __fma_rn(wz[3], c3, __fma_rn(wz[2], c2, __fma_rn(wz[1], c1, wz[0] * c0)));
        t[0][e] = __fma_rn(wy[J], s0, t[0][e]);
        if (KIND != SPO_KIND_V) {
            const double s1 = __fma_rn(wz[7], c3, __fma_rn(wz[6], c2, __fma_rn(wz[5], c1, wz[4] * c0)));
            const double s2 = __fma_rn(wz[11], c3, __fma_rn(wz[10], c2, __fma_rn(wz[9], c1, wz[8] * c0)));
            t[1][e] = __fma_rn(wy[4 + J], s0, t[1][e]);
            t[2][e] = __fma_rn(wy[J], s1, t[2][e]);
            t[3][e] = __fma_rn(wy[8 + J], s0, t[3][e]);
            t[5][e] = __fma_rn(wy[J], s2, t[5][e]);
            if (KIND == SPO_KIND_VGH) t[4][e] = __fma_rn(wy[4 + J], s1, t[4][e]);
        }
    }
}
template <int KIND>
__device__ __forceinline__ void slab_done(double ax, double dax, double d2ax, const double (&t)[6][2],
                                          double2 (&acc)[NS<KIND>::S][1]) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        double *a0 = e ? &acc[0][0].y : &acc[0][0].x;
        *a0 = __fma_rn(ax, t[0][e], *a0);
        if (KIND != SPO_KIND_V) {
            double *a1 = e ? &acc[1][0].y : &acc[1][0].x;
            double *a2 = e ? &acc[2][0].y : &acc[2][0].x;
            double *a3 = e ? &acc[3][0].y : &acc[3][0].x;
            *a1 = __fma_rn(dax, t[0][e], *a1);
            *a2 = __fma_rn(ax, t[1][e], *a2);
            *a3 = __fma_rn(ax, t[2][e], *a3);
        }
        if (KIND == SPO_KIND_VGL) {
            double *a4 = e ? &acc[4][0].y : &acc[4][0].x;
            *a4 = __fma_rn(d2ax, t[0][e], __fma_rn(ax, t[3][e], __fma_rn(ax, t[5][e], *a4)));
        }
        if (KIND == SPO_KIND_VGH) {
            double *a4 = e ? &acc[4][0].y : &acc[4][0].x;
            double *a5 = e ? &acc[5][0].y : &acc[5][0].x;
            double *a6 = e ? &acc[6][0].y : &acc[6][0].x;
            double *a7 = e ? &acc[7][0].y : &acc[7][0].x;
            double *a8 = e ? &acc[8][0].y : &acc[8][0].x;
            double *a9 = e ? &acc[9][0].y : &acc[9][0].x;
            *a4 = __fma_rn(d2ax, t[0][e], *a4);
            *a5 = __fma_rn(dax, t[1][e], *a5);
            *a6 = __fma_rn(dax, t[2][e], *a6);
            *a7 = __fma_rn(ax, t[3][e], *a7);
            *a8 = __fma_rn(ax, t[4][e], *a8);
            *a9 = __fma_rn(ax, t[5][e], *a9);
        }
    }
}
template <int KIND, int CW, int RJ = 4>
__device__ __forceinline__ void slab_contract(const double *__restrict__ slab, const double (&wy)[12],
                                              const double (&wz)[12], double ax, double dax, double d2ax,
                                              double2 (&acc)[NS<KIND>::S][1]) {
    double t[6][2];
#pragma unroll
    for (int u = 0; u < 6; ++u) t[u][0] = t[u][1] = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        double2 c[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) c[k] = *reinterpret_cast<const double2 *>(slab + (j * RJ + k) * CW);
        if (j == 0) rowgroup<KIND, 0>(c, wy, wz, t);
        if (j == 1) rowgroup<KIND, 1>(c, wy, wz, t);
        if (j == 2) rowgroup<KIND, 2>(c, wy, wz, t);
        if (j == 3) rowgroup<KIND, 3>(c, wy, wz, t);
    }
    slab_done<KIND>(ax, dax, d2ax, t, acc);
}

// ---- k-power form (SPO_FORM_KPOWER tables): the 4 rows of (i, j) hold the
// power-basis coefficients q0..q3 of the cubic along k, so that
//   sum_k a_k(t) c_k   = q0 + t q1 + t^2 q2 + t^3 q3            (= A)
//   sum_k da_k/dt c_k  = q1 + 2t q2 + 3t^2 q3                   (= D)
//   sum_k d2a_k/dt2 c_k / 2 = q2 + 3t q3                        (= H)
// with a_k the uniform cubic B-spline basis of grid.py:127-130.  Seven packed
// FMAs per (i, j) row group give all three k-sums (the B-spline form needs
// twelve), and the only z weight is t itself.  The 1/dz and 2/dz^2 factors of
// D and H are folded into the x weights of the streams that use them (axz =
// ax/dz, daxz = dax/dz, axz2 = 2 ax/dz^2).
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }

template <int KIND>
__device__ __forceinline__ void kpow_sums(float t, float2 q0, float2 q1, float2 q2, float2 q3, float2 &A, float2 &D,
                                          float2 &H) {
    const float2 e = fma2(t, q3, q2);  // q2 + t q3
    A = fma2(t, fma2(t, e, q1), q0);
    if (KIND != SPO_KIND_V) {
        const float2 h = fma2(t, q3, e);  // q2 + 2t q3
        D = fma2(t, add2(e, h), q1);      // q1 + t (2 q2 + 3t q3)
        H = fma2(t, q3, h);               // q2 + 3t q3
    }
}
template <int KIND>
__device__ __forceinline__ void kpow_sums(double t, double q0, double q1, double q2, double q3, double &A, double &D,
                                          double &H) {
    const double e = __fma_rn(t, q3, q2);
    A = __fma_rn(t, __fma_rn(t, e, q1), q0);
    if (KIND != SPO_KIND_V) {
        const double h = __fma_rn(t, q3, e);
        D = __fma_rn(t, __dadd_rn(e, h), q1);
        H = __fma_rn(t, q3, h);
    }
}

// One i-slab of a k-power table for one lane (4 fp32 orbitals).
template <int KIND, int CW>
__device__ __forceinline__ void slab_contract_kp(const float *__restrict__ slab, const float (&wy)[12], float tz,
                                                 float ax, float dax, float d2ax, float axz, float daxz, float axz2,
                                                 float2 (&acc)[NS<KIND>::S][2]) {
    float2 t00[2], t10[2], t01[2], t20[2], t11[2], t02[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) t00[h] = t10[h] = t01[h] = t20[h] = t11[h] = t02[h] = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        float4 c[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) c[k] = *reinterpret_cast<const float4 *>(slab + (j * 4 + k) * CW);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float2 q0 = h ? make_float2(c[0].z, c[0].w) : make_float2(c[0].x, c[0].y);
            const float2 q1 = h ? make_float2(c[1].z, c[1].w) : make_float2(c[1].x, c[1].y);
            const float2 q2 = h ? make_float2(c[2].z, c[2].w) : make_float2(c[2].x, c[2].y);
            const float2 q3 = h ? make_float2(c[3].z, c[3].w) : make_float2(c[3].x, c[3].y);
            float2 A, D, H;
            kpow_sums<KIND>(tz, q0, q1, q2, q3, A, D, H);
            t00[h] = fma2(wy[j], A, t00[h]);
            if (KIND != SPO_KIND_V) {
                t10[h] = fma2(wy[4 + j], A, t10[h]);
                t01[h] = fma2(wy[j], D, t01[h]);
                t20[h] = fma2(wy[8 + j], A, t20[h]);
                t02[h] = fma2(wy[j], H, t02[h]);
                if (KIND == SPO_KIND_VGH) t11[h] = fma2(wy[4 + j], D, t11[h]);
            }
        }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        acc[0][h] = fma2(ax, t00[h], acc[0][h]);
        if (KIND != SPO_KIND_V) {
            acc[1][h] = fma2(dax, t00[h], acc[1][h]);
            acc[2][h] = fma2(ax, t10[h], acc[2][h]);
            acc[3][h] = fma2(axz, t01[h], acc[3][h]);
        }
        if (KIND == SPO_KIND_VGL) acc[4][h] = fma2(d2ax, t00[h], fma2(ax, t20[h], fma2(axz2, t02[h], acc[4][h])));
        if (KIND == SPO_KIND_VGH) {
            acc[4][h] = fma2(d2ax, t00[h], acc[4][h]);
            acc[5][h] = fma2(dax, t10[h], acc[5][h]);
            acc[6][h] = fma2(daxz, t01[h], acc[6][h]);
            acc[7][h] = fma2(ax, t20[h], acc[7][h]);
            acc[8][h] = fma2(axz, t11[h], acc[8][h]);
            acc[9][h] = fma2(axz2, t02[h], acc[9][h]);
        }
    }
}

// One i-slab of a k-power table for one lane (2 fp64 orbitals).
template <int KIND, int CW>
__device__ __forceinline__ void slab_contract_kp(const double *__restrict__ slab, const double (&wy)[12], double tz,
                                                 double ax, double dax, double d2ax, double axz, double daxz,
                                                 double axz2, double2 (&acc)[NS<KIND>::S][1]) {
    double t00[2], t10[2], t01[2], t20[2], t11[2], t02[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) t00[e] = t10[e] = t01[e] = t20[e] = t11[e] = t02[e] = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        double2 c[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) c[k] = *reinterpret_cast<const double2 *>(slab + (j * 4 + k) * CW);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            double A, D, H;
            kpow_sums<KIND>(tz, e ? c[0].y : c[0].x, e ? c[1].y : c[1].x, e ? c[2].y : c[2].x, e ? c[3].y : c[3].x,
                            A, D, H);
            t00[e] = __fma_rn(wy[j], A, t00[e]);
            if (KIND != SPO_KIND_V) {
                t10[e] = __fma_rn(wy[4 + j], A, t10[e]);
                t01[e] = __fma_rn(wy[j], D, t01[e]);
                t20[e] = __fma_rn(wy[8 + j], A, t20[e]);
                t02[e] = __fma_rn(wy[j], H, t02[e]);
                if (KIND == SPO_KIND_VGH) t11[e] = __fma_rn(wy[4 + j], D, t11[e]);
            }
        }
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        double *a0 = e ? &acc[0][0].y : &acc[0][0].x;
        *a0 = __fma_rn(ax, t00[e], *a0);
        if (KIND != SPO_KIND_V) {
            double *a1 = e ? &acc[1][0].y : &acc[1][0].x;
            double *a2 = e ? &acc[2][0].y : &acc[2][0].x;
            double *a3 = e ? &acc[3][0].y : &acc[3][0].x;
            *a1 = __fma_rn(dax, t00[e], *a1);
            *a2 = __fma_rn(ax, t10[e], *a2);
            *a3 = __fma_rn(axz, t01[e], *a3);
        }
        if (KIND == SPO_KIND_VGL) {
            double *a4 = e ? &acc[4][0].y : &acc[4][0].x;
            *a4 = __fma_rn(d2ax, t00[e], __fma_rn(ax, t20[e], __fma_rn(axz2, t02[e], *a4)));
        }
        if (KIND == SPO_KIND_VGH) {
            double *a4 = e ? &acc[4][0].y : &acc[4][0].x;
            double *a5 = e ? &acc[5][0].y : &acc[5][0].x;
            double *a6 = e ? &acc[6][0].y : &acc[6][0].x;
            double *a7 = e ? &acc[7][0].y : &acc[7][0].x;
            double *a8 = e ? &acc[8][0].y : &acc[8][0].x;
            double *a9 = e ? &acc[9][0].y : &acc[9][0].x;
            *a4 = __fma_rn(d2ax, t00[e], *a4);
            *a5 = __fma_rn(dax, t10[e], *a5);
            *a6 = __fma_rn(daxz, t01[e], *a6);
            *a7 = __fma_rn(ax, t20[e], *a7);
            *a8 = __fma_rn(axz, t11[e], *a8);
            *a9 = __fma_rn(axz2, t02[e], *a9);
        }
    }
}

// ---- V, several positions per consumer warp (the line kernel's VGROUP
// path): one row group (the 4 k-rows of one j) of a plane contracted for one
// position into its per-plane j-sum t00 -- exactly the V sequence of
// slab_contract / slab_contract_kp (bitwise), so a plane's rows are read from
// shared memory once for every position of the group that covers the plane.
template <bool KP>
__device__ __forceinline__ void v_rowgroup(const float4 (&c)[4], const float (&wz)[4], float wyj, float2 (&t00)[2]) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const float2 c0 = h ? make_float2(c[0].z, c[0].w) : make_float2(c[0].x, c[0].y);
        const float2 c1 = h ? make_float2(c[1].z, c[1].w) : make_float2(c[1].x, c[1].y);
        const float2 c2 = h ? make_float2(c[2].z, c[2].w) : make_float2(c[2].x, c[2].y);
        const float2 c3 = h ? make_float2(c[3].z, c[3].w) : make_float2(c[3].x, c[3].y);
        float2 s0, d, hh;
        if constexpr (KP)
            kpow_sums<SPO_KIND_V>(wz[0], c0, c1, c2, c3, s0, d, hh);
        else
            s0 = fma2(wz[3], c3, fma2(wz[2], c2, fma2(wz[1], c1, mul2(wz[0], c0))));
        t00[h] = fma2(wyj, s0, t00[h]);
    }
}
template <bool KP>
__device__ __forceinline__ void v_rowgroup(const double2 (&c)[4], const double (&wz)[4], double wyj,
                                           double (&t00)[2]) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const double c0 = e ? c[0].y : c[0].x, c1 = e ? c[1].y : c[1].x;
        const double c2 = e ? c[2].y : c[2].x, c3 = e ? c[3].y : c[3].x;
        double s0, d, hh;
        if constexpr (KP)
            kpow_sums<SPO_KIND_V>(wz[0], c0, c1, c2, c3, s0, d, hh);
        else
            s0 = __fma_rn(wz[3], c3, __fma_rn(wz[2], c2, __fma_rn(wz[1], c1, wz[0] * c0)));
        t00[e] = __fma_rn(wyj, s0, t00[e]);
    }
}
__device__ __forceinline__ void v_plane_done(float ax, float2 (&t00)[2], float2 (&acc)[1][2]) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        acc[0][h] = fma2(ax, t00[h], acc[0][h]);
        t00[h] = make_float2(0.f, 0.f);
    }
}
__device__ __forceinline__ void v_plane_done(double ax, double (&t00)[2], double2 (&acc)[1][1]) {
    acc[0][0].x = __fma_rn(ax, t00[0], acc[0][0].x);
    acc[0][0].y = __fma_rn(ax, t00[1], acc[0][0].y);
    t00[0] = t00[1] = 0.0;
}
__device__ __forceinline__ void load4(const unsigned char *p, float (&w)[4]) {
    const float4 v = *reinterpret_cast<const float4 *>(p);
    w[0] = v.x, w[1] = v.y, w[2] = v.z, w[3] = v.w;
}
__device__ __forceinline__ void load4(const unsigned char *p, double (&w)[4]) {
    const double2 v0 = reinterpret_cast<const double2 *>(p)[0], v1 = reinterpret_cast<const double2 *>(p)[1];
    w[0] = v0.x, w[1] = v0.y, w[2] = v1.x, w[3] = v1.y;
}

// The 36 weights of a record (16-byte aligned in shared memory) as 16-byte
// loads: 9 (fp32) / 18 (fp64) LDS.128 instead of 36 scalar LDS -- uniform
// addresses, one wavefront each.  Unused weights (k-power tables read only
// wz[0]) are dropped by the compiler.
__device__ __forceinline__ void load_weights(const unsigned char *rec, float (&wx)[12], float (&wy)[12],
                                             float (&wz)[12]) {
    const float4 *q = reinterpret_cast<const float4 *>(rec);
#pragma unroll
    for (int v = 0; v < 3; ++v) {
        const float4 a = q[v], b = q[3 + v], c = q[6 + v];
        wx[4 * v] = a.x, wx[4 * v + 1] = a.y, wx[4 * v + 2] = a.z, wx[4 * v + 3] = a.w;
        wy[4 * v] = b.x, wy[4 * v + 1] = b.y, wy[4 * v + 2] = b.z, wy[4 * v + 3] = b.w;
        wz[4 * v] = c.x, wz[4 * v + 1] = c.y, wz[4 * v + 2] = c.z, wz[4 * v + 3] = c.w;
    }
}
__device__ __forceinline__ void load_weights(const unsigned char *rec, double (&wx)[12], double (&wy)[12],
                                             double (&wz)[12]) {
    const double2 *q = reinterpret_cast<const double2 *>(rec);
#pragma unroll
    for (int v = 0; v < 6; ++v) {
        const double2 a = q[v], b = q[6 + v], c = q[12 + v];
        wx[2 * v] = a.x, wx[2 * v + 1] = a.y;
        wy[2 * v] = b.x, wy[2 * v + 1] = b.y;
        wz[2 * v] = c.x, wz[2 * v + 1] = c.y;
    }
}

template <typename T>
struct Acc;
template <>
struct Acc<float> {
    using V = float2;
    static constexpr int N = 2;  // two fp32x2 pairs = the lane's 4 orbitals
};
template <>
struct Acc<double> {
    using V = double2;
    static constexpr int N = 1;  // one pair = the lane's 2 orbitals
};

__device__ __forceinline__ void zero(float2 &v) { v = make_float2(0.f, 0.f); }
__device__ __forceinline__ void zero(double2 &v) { v = make_double2(0.0, 0.0); }

template <int S>
__device__ __forceinline__ void store_lane(float *o, long long sstride, const float2 (&acc)[S][2], bool finite) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const float4 v = finite ? make_float4(acc[s][0].x, acc[s][0].y, acc[s][1].x, acc[s][1].y)
                                : make_float4(NAN, NAN, NAN, NAN);
        __stcs(reinterpret_cast<float4 *>(o + s * sstride), v);
    }
}
template <int S>
__device__ __forceinline__ void store_lane(double *o, long long sstride, const double2 (&acc)[S][1], bool finite) {
#pragma unroll
    for (int s = 0; s < S; ++s)
        __stcs(reinterpret_cast<double2 *>(o + s * sstride), finite ? acc[s][0] : make_double2(NAN, NAN));
}
// the lane vector straddles lane_limit: store its first `nv` lanes only
// (unrolled + predicated: no dynamic indexing of the accumulators)
template <int S>
__device__ __forceinline__ void store_lane_partial(float *o, long long sstride, const float2 (&acc)[S][2],
                                                   bool finite, int nv) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
        if (nv > 0) o[s * sstride + 0] = finite ? acc[s][0].x : NAN;
        if (nv > 1) o[s * sstride + 1] = finite ? acc[s][0].y : NAN;
        if (nv > 2) o[s * sstride + 2] = finite ? acc[s][1].x : NAN;
    }
}
template <int S>
__device__ __forceinline__ void store_lane_partial(double *o, long long sstride, const double2 (&acc)[S][1],
                                                   bool finite, int nv) {
#pragma unroll
    for (int s = 0; s < S; ++s)
        if (nv > 0) o[s * sstride] = finite ? acc[s][0].x : NAN;
}

// Fused epilogue: this lane's orbitals dotted with its coefficient entries in
// fp64, reduced over the LPP lanes of the position (xor shuffles stay inside
// the lane segment), written once per (unit, position) by the segment leader.
// fp32 tables: the lane's 4-term dot and the lane-segment reduction run in
// fp32 (one chunk = at most 128 orbitals); chunks are summed in fp64.
template <int S, int LPP>
__device__ __forceinline__ void ratio_partials(const float2 (&acc)[S][2], const float *coef, bool live,
                                               double (&part)[S]) {
    float4 cf = make_float4(0.f, 0.f, 0.f, 0.f);
    if (live) cf = __ldg(reinterpret_cast<const float4 *>(coef));
    float f[S];
#pragma unroll
    for (int s = 0; s < S; ++s)
        f[s] = live ? __fmaf_rn(acc[s][1].y, cf.w,
                                __fmaf_rn(acc[s][1].x, cf.z, __fmaf_rn(acc[s][0].y, cf.y, acc[s][0].x * cf.x)))
                    : 0.0f;
#pragma unroll
    for (int off = LPP / 2; off > 0; off >>= 1)
#pragma unroll
        for (int s = 0; s < S; ++s) f[s] += __shfl_xor_sync(0xffffffffu, f[s], off);
#pragma unroll
    for (int s = 0; s < S; ++s) part[s] = f[s];
}
template <int S, int LPP>
__device__ __forceinline__ void ratio_partials(const double2 (&acc)[S][1], const double *coef, bool live,
                                               double (&part)[S]) {
    double2 cf = make_double2(0.0, 0.0);
    if (live) cf = __ldg(reinterpret_cast<const double2 *>(coef));
#pragma unroll
    for (int s = 0; s < S; ++s) part[s] = live ? __fma_rn(acc[s][0].y, cf.y, acc[s][0].x * cf.x) : 0.0;
#pragma unroll
    for (int off = LPP / 2; off > 0; off >>= 1)
#pragma unroll
        for (int s = 0; s < S; ++s) part[s] += __shfl_xor_sync(0xffffffffu, part[s], off);
}

}  // namespace tma
}  // namespace spo

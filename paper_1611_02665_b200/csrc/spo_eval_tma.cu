// spo_eval_tma.cu -- TMA-pipelined V / VGL / VGH kernels (the fast path, fp32
// and fp64).
//
// Same math as spo_eval.cu's separable FAST contraction (kernels.py:143-247
// restated as k-, then j-, then i-sums with FMA, bitwise the same sequence),
// different data movement:
//
//  1. bucket_count_kernel + prologue_records_kernel: one thread per position
//     maps it to (i0,j0,k0) and its 36 basis weights (fp32: bit-exact grid.py
//     form; fp64: oracle.py form) into a record carrying the cell and the
//     original index, counting-sorted into 4x4x4 spatial blocks of the grid.
//  2. eval_tma_kernel: persistent CTAs (one per SM).  Work items are (unit u =
//     (tile m, chunk c of CW lanes), batch of BP bucket-sorted positions),
//     handed out by a global ticket counter in unit-major order, so at any
//     moment the GPU works on one CW-wide slice of the table and, inside it,
//     on one spatial block: the L2 working set is a block's rows x CW lanes
//     (2.4 MB for 67^3 at 128 fp32 lanes) -- the paper's AoSoA cache blocking,
//     enforced by scheduling.
//     Per warp, a 2-stage ring of 8 KB shared-memory stages is fed by TMA: one
//     cp.async.bulk.tensor.5d per (position, i) brings the 4(j) x 4(k) x CW
//     slab (16 rows) and completes on the stage's mbarrier; item records
//     arrive by cp.async.bulk on their own mbarriers (double-buffered).  The
//     warp issues one slab ahead of its compute, across group/item bounds.
//     Compute: lane = (position in group, 16-byte lane vector: 4 fp32 / 2 fp64
//     orbitals), S accumulators per orbital in registers over the 4 i-slabs;
//     fp32 FMAs as packed FFMA2, fp64 as DFMA; 16-byte streaming stores.
#include <cuda.h>

#include <cstdlib>

#include "spo_common.cuh"
#include "spo_prologue.cuh"

namespace spo {
namespace tma {

constexpr int STAGE = 8192;      // bytes: 32 lanes x 16 B x 16 rows
constexpr int WS_HEADER = 1024;  // ticket @0, bucket counts @256, bucket cursors @512

// Launch shapes: warps per CTA, ring stages per warp, positions per item.
template <int WARPS_, int R_, int BP_>
struct TCfg {
    static constexpr int WARPS = WARPS_, R = R_, BP = BP_;
};

template <typename T>
struct TT;
template <>
struct TT<float> {
    static constexpr int W = 4;                   // elements per 16-byte lane vector
    static constexpr int RECB = 36 * 4 + 16;      // record bytes: 36 weights + i0 j0 k0 orig
    using Cfg = TCfg<12, 2, 8>;                   // 160 registers per thread
};
template <>
struct TT<double> {
    static constexpr int W = 2;
    static constexpr int RECB = 36 * 8 + 16;
    // fp64 weights need ~200 registers: 8 warps (2 per SMSP register-file
    // partition) instead of 12 (3 per partition would cap them at 168)
    using Cfg = TCfg<8, 2, 8>;
};

struct Args {
    const unsigned char *recs;  // [n_pos][RECB] bucket-sorted
    unsigned *ticket;
    long long n_pos;
    long long nbatch;           // ceil(n_pos / bp)
    int bp;                     // positions per item (<= BP; small batches use fewer)
    long long n_items;          // units * nbatch
    int chunks;                 // chunks of CW lanes per tile row
    int nb;                     // table row length (lanes)
    void *out;
    long long out_pos_stride, out_stream_stride;
    const long long *out_index;
    long long lane_limit;       // output lanes >= lane_limit are not stored
    int evict_last;             // L2 evict_last hint on table slabs
    int proxy_fence;            // fence.proxy.async before reusing a stage (diagnostic)
    // fused ratio epilogue (RATIO kernels): per (unit, position) partial dot
    // products of every stream with the caller's coefficient row
    const void *coef;           // [n_pos][coef_stride] in output-lane layout, pad lanes 0
    long long coef_stride;
    double *partials;           // [units][n_pos][S]
};

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
// slab: [j][k][CW] of this lane's position; wy/wz: 12 weights; ax/dax/d2ax: x weights of this i.
template <int KIND, int CW>
__device__ __forceinline__ void slab_contract(const float *__restrict__ slab, const float (&wy)[12],
                                              const float (&wz)[12], float ax, float dax, float d2ax,
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
            const float2 c0 = h ? make_float2(c[0].z, c[0].w) : make_float2(c[0].x, c[0].y);
            const float2 c1 = h ? make_float2(c[1].z, c[1].w) : make_float2(c[1].x, c[1].y);
            const float2 c2 = h ? make_float2(c[2].z, c[2].w) : make_float2(c[2].x, c[2].y);
            const float2 c3 = h ? make_float2(c[3].z, c[3].w) : make_float2(c[3].x, c[3].y);
            const float2 s0 = fma2(wz[3], c3, fma2(wz[2], c2, fma2(wz[1], c1, mul2(wz[0], c0))));
            t00[h] = fma2(wy[j], s0, t00[h]);
            if (KIND != SPO_KIND_V) {
                const float2 s1 = fma2(wz[7], c3, fma2(wz[6], c2, fma2(wz[5], c1, mul2(wz[4], c0))));
                const float2 s2 = fma2(wz[11], c3, fma2(wz[10], c2, fma2(wz[9], c1, mul2(wz[8], c0))));
                t10[h] = fma2(wy[4 + j], s0, t10[h]);
                t01[h] = fma2(wy[j], s1, t01[h]);
                t20[h] = fma2(wy[8 + j], s0, t20[h]);
                t02[h] = fma2(wy[j], s2, t02[h]);
                if (KIND == SPO_KIND_VGH) t11[h] = fma2(wy[4 + j], s1, t11[h]);
            }
        }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        acc[0][h] = fma2(ax, t00[h], acc[0][h]);
        if (KIND != SPO_KIND_V) {
            acc[1][h] = fma2(dax, t00[h], acc[1][h]);
            acc[2][h] = fma2(ax, t10[h], acc[2][h]);
            acc[3][h] = fma2(ax, t01[h], acc[3][h]);
        }
        if (KIND == SPO_KIND_VGL) acc[4][h] = fma2(d2ax, t00[h], fma2(ax, t20[h], fma2(ax, t02[h], acc[4][h])));
        if (KIND == SPO_KIND_VGH) {
            acc[4][h] = fma2(d2ax, t00[h], acc[4][h]);
            acc[5][h] = fma2(dax, t10[h], acc[5][h]);
            acc[6][h] = fma2(dax, t01[h], acc[6][h]);
            acc[7][h] = fma2(ax, t20[h], acc[7][h]);
            acc[8][h] = fma2(ax, t11[h], acc[8][h]);
            acc[9][h] = fma2(ax, t02[h], acc[9][h]);
        }
    }
}

// One i-slab for one lane: 2 fp64 orbitals, DFMA in the generic kernel's order.
template <int KIND, int CW>
__device__ __forceinline__ void slab_contract(const double *__restrict__ slab, const double (&wy)[12],
                                              const double (&wz)[12], double ax, double dax, double d2ax,
                                              double2 (&acc)[NS<KIND>::S][1]) {
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
            const double c0 = e ? c[0].y : c[0].x, c1 = e ? c[1].y : c[1].x;
            const double c2 = e ? c[2].y : c[2].x, c3 = e ? c[3].y : c[3].x;
            const double s0 = __fma_rn(wz[3], c3, __fma_rn(wz[2], c2, __fma_rn(wz[1], c1, wz[0] * c0)));
            t00[e] = __fma_rn(wy[j], s0, t00[e]);
            if (KIND != SPO_KIND_V) {
                const double s1 = __fma_rn(wz[7], c3, __fma_rn(wz[6], c2, __fma_rn(wz[5], c1, wz[4] * c0)));
                const double s2 = __fma_rn(wz[11], c3, __fma_rn(wz[10], c2, __fma_rn(wz[9], c1, wz[8] * c0)));
                t10[e] = __fma_rn(wy[4 + j], s0, t10[e]);
                t01[e] = __fma_rn(wy[j], s1, t01[e]);
                t20[e] = __fma_rn(wy[8 + j], s0, t20[e]);
                t02[e] = __fma_rn(wy[j], s2, t02[e]);
                if (KIND == SPO_KIND_VGH) t11[e] = __fma_rn(wy[4 + j], s1, t11[e]);
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
            *a3 = __fma_rn(ax, t01[e], *a3);
        }
        if (KIND == SPO_KIND_VGL) {
            double *a4 = e ? &acc[4][0].y : &acc[4][0].x;
            *a4 = __fma_rn(d2ax, t00[e], __fma_rn(ax, t20[e], __fma_rn(ax, t02[e], *a4)));
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
            *a6 = __fma_rn(dax, t01[e], *a6);
            *a7 = __fma_rn(ax, t20[e], *a7);
            *a8 = __fma_rn(ax, t11[e], *a8);
            *a9 = __fma_rn(ax, t02[e], *a9);
        }
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

// ------------------------------------------------------------ prologue --
// Positions are binned by the spatial block (NBK^3 blocks of the grid) of
// their stencil cell, so that the eval kernel's unit-major sweep touches one
// block's rows at a time: the L2 working set is (rows / NBK^3) x CW lanes,
// small enough for 512-byte chunks (one TMA per position-slab).
constexpr int NBK = 4;
constexpr int NBUCKET = NBK * NBK * NBK;

__device__ __forceinline__ int bucket_of_cell(int i0, int j0, int k0, const GridArgs &g) {
    if (i0 < 0) return 0;
    const int bi = i0 * NBK / g.n[0], bj = j0 * NBK / g.n[1], bk = k0 * NBK / g.n[2];
    return (bi * NBK + bj) * NBK + bk;
}

// pass 1: bucket of every position + bucket histogram (block-aggregated)
__global__ void bucket_count_kernel(GridArgs g, const double *__restrict__ pos, long long n,
                                    unsigned char *__restrict__ bucket, unsigned *__restrict__ counts) {
    __shared__ unsigned hist[NBUCKET];
    for (int b = threadIdx.x; b < NBUCKET; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
         p += (long long)gridDim.x * blockDim.x) {
        double t;
        const double x = pos[3 * p], y = pos[3 * p + 1], z = pos[3 * p + 2];
        int i0 = map_axis(x, g.dinv[0], g.cnt[0], &t);
        const int j0 = map_axis(y, g.dinv[1], g.cnt[1], &t);
        const int k0 = map_axis(z, g.dinv[2], g.cnt[2], &t);
        if (!(isfinite(x) && isfinite(y) && isfinite(z))) i0 = -1;
        const int b = bucket_of_cell(i0, j0, k0, g);
        bucket[p] = (unsigned char)b;
        atomicAdd(&hist[b], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < NBUCKET; b += blockDim.x)
        if (hist[b]) atomicAdd(&counts[b], hist[b]);
}

__device__ __forceinline__ void store_weights(unsigned char *dst, const float (&w)[36]) {
#pragma unroll
    for (int e = 0; e < 9; ++e)
        reinterpret_cast<float4 *>(dst)[e] = make_float4(w[4 * e], w[4 * e + 1], w[4 * e + 2], w[4 * e + 3]);
}
__device__ __forceinline__ void store_weights(unsigned char *dst, const double (&w)[36]) {
#pragma unroll
    for (int e = 0; e < 18; ++e) reinterpret_cast<double2 *>(dst)[e] = make_double2(w[2 * e], w[2 * e + 1]);
}

// pass 2: records (bit-exact mapping + 36 weights + cell + original index)
// scattered to their bucket's range; slots are reserved per block.
template <typename T>
__global__ void prologue_records_kernel(GridArgs g, const double *__restrict__ pos, long long n,
                                        const unsigned char *__restrict__ bucket,
                                        const unsigned *__restrict__ counts, unsigned *__restrict__ cursors,
                                        unsigned char *__restrict__ recs, int *__restrict__ status) {
    constexpr int RECB = TT<T>::RECB;
    __shared__ unsigned offs[NBUCKET], local[NBUCKET], base[NBUCKET];
    if (threadIdx.x == 0) {
        unsigned s = 0;
        for (int b = 0; b < NBUCKET; ++b) {
            offs[b] = s;
            s += counts[b];
        }
    }
    for (long long p0 = blockIdx.x * (long long)blockDim.x; p0 < n; p0 += (long long)gridDim.x * blockDim.x) {
        const long long p = p0 + threadIdx.x;
        for (int b = threadIdx.x; b < NBUCKET; b += blockDim.x) local[b] = 0;
        __syncthreads();
        const int b = p < n ? bucket[p] : 0;
        const unsigned rank = p < n ? atomicAdd(&local[b], 1u) : 0u;
        __syncthreads();
        for (int q = threadIdx.x; q < NBUCKET; q += blockDim.x)
            base[q] = local[q] ? offs[q] + atomicAdd(&cursors[q], local[q]) : 0u;
        __syncthreads();
        if (p < n) {
            const double x = pos[3 * p], y = pos[3 * p + 1], z = pos[3 * p + 2];
            double tx, ty, tz;
            int i0 = map_axis(x, g.dinv[0], g.cnt[0], &tx);
            const int j0 = map_axis(y, g.dinv[1], g.cnt[1], &ty);
            const int k0 = map_axis(z, g.dinv[2], g.cnt[2], &tz);
            T w[36];
            axis_weights<T>(tx, g.dinv[0], g.delta[0], w);
            axis_weights<T>(ty, g.dinv[1], g.delta[1], w + 12);
            axis_weights<T>(tz, g.dinv[2], g.delta[2], w + 24);
            if (!(isfinite(x) && isfinite(y) && isfinite(z))) {
                if (status) atomicOr(status, 1);
                i0 = -1;
            }
            unsigned char *dst = recs + (long long)(base[b] + rank) * RECB;
            store_weights(dst, w);
            *reinterpret_cast<int4 *>(dst + 36 * sizeof(T)) = make_int4(i0, j0, k0, (int)p);
        }
        __syncthreads();
    }
}

// -------------------------------------------------------------- kernel --
struct ItemInfo {
    long long b0;
    int nb, m, c, G, valid, pad;
};

// Issue descriptor of one group (lane 0's registers): per position the
// TMA coordinates and whether it is valid; the chunk/tile of the item.
template <int PW>
struct GroupDesc {
    int x[PW], y[PW], z[PW];  // i0, j0, k0 (z = k0 is the fastest table dim after lanes)
    unsigned bytes;           // valid positions x slab bytes
    int c0, m;
};

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

template <int KIND, typename T, int CW, class C, bool RATIO>
__global__ void __launch_bounds__(C::WARPS * 32, 1)
    eval_tma_kernel(const __grid_constant__ CUtensorMap tmap, const Args a) {
    constexpr int WARPS = C::WARPS, BP = C::BP;
    static_assert(C::R == 2, "the issue path runs exactly one slab ahead");
    constexpr int R = 2;
    constexpr int S = NS<KIND>::S;
    constexpr int W = TT<T>::W;
    constexpr int RECB = TT<T>::RECB;
    constexpr int PW = 32 * W / CW;              // positions per warp step
    constexpr int LPP = CW / W;                  // lanes per position
    constexpr int SLAB = CW * 16 * sizeof(T);    // bytes per (position, i) slab
    using AV = typename Acc<T>::V;
    constexpr int AN = Acc<T>::N;
    static_assert(PW * SLAB == STAGE, "stage must hold one warp step");
    static_assert(BP % PW == 0, "items hold whole groups");

    extern __shared__ __align__(1024) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char *ring = smem + (size_t)warp * R * STAGE;
    unsigned long long *bars =
        reinterpret_cast<unsigned long long *>(smem + (size_t)WARPS * R * STAGE) + warp * (R + 2);
    unsigned long long *rbar = bars + R;  // record barriers of slots 0/1
    unsigned char *recs = smem + (size_t)WARPS * R * STAGE + WARPS * (R + 2) * 8 + (size_t)warp * 2 * BP * RECB;
    ItemInfo *info = reinterpret_cast<ItemInfo *>(smem + (size_t)WARPS * R * STAGE + WARPS * (R + 2) * 8 +
                                                  (size_t)WARPS * 2 * BP * RECB) + warp * 2;

    if (lane == 0) {
        for (int s = 0; s < R + 2; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();

    // Take a ticket and start the record copy of its item into `slot`.
    auto fill = [&](int slot) {
        if (lane == 0) {
            const unsigned long long k = atomicAdd(a.ticket, 1u);
            ItemInfo it;
            it.valid = k < (unsigned long long)a.n_items;
            if (it.valid) {
                const long long u = (long long)k / a.nbatch;
                const long long b = (long long)k - u * a.nbatch;
                it.m = (int)(u / a.chunks);
                it.c = (int)(u - (long long)it.m * a.chunks);
                it.b0 = b * a.bp;
                it.nb = (int)min((long long)a.bp, a.n_pos - it.b0);
                it.G = (it.nb + PW - 1) / PW;
                if (a.proxy_fence) fence_proxy_async();  // WAR on the slot, see issue()
                mbar_arrive_expect_tx(&rbar[slot], (unsigned)(it.nb * RECB));
                bulk_load(recs + slot * BP * RECB, a.recs + it.b0 * RECB, (unsigned)(it.nb * RECB), &rbar[slot]);
            } else {
                it.b0 = 0;
                it.nb = it.m = it.c = it.G = 0;
            }
            info[slot] = it;
        }
        __syncwarp();
    };

    // lane 0: descriptor of group g of the item in `slot` (records must have landed)
    auto prepare = [&](GroupDesc<PW> &d, int slot, int g) {
        const ItemInfo it = info[slot];
        const unsigned char *rc = recs + slot * BP * RECB;
        d.bytes = 0;
        d.c0 = it.c * CW;
        d.m = it.m;
#pragma unroll
        for (int q = 0; q < PW; ++q) {
            const int p = g * PW + q;
            const int4 cell = *reinterpret_cast<const int4 *>(rc + min(p, it.nb - 1) * RECB + 36 * sizeof(T));
            const bool ok = p < it.nb && cell.x >= 0;
            d.x[q] = ok ? cell.x : -1;
            d.y[q] = cell.y;
            d.z[q] = cell.z;
            d.bytes += ok ? SLAB : 0;
        }
    };
    // lane 0: issue slab ii of the described group into stage st
    auto issue = [&](const GroupDesc<PW> &d, int ii, int st, unsigned long long policy) {
        unsigned char *dst = ring + st * STAGE;
        // WAR only (LDS reads of this stage, all consumed before the
        // __syncwarp before this call, then the TMA write): no proxy fence
        // needed, as in a consumer-release / producer-acquire TMA pipeline.
        if (a.proxy_fence) fence_proxy_async();
        mbar_arrive_expect_tx(&bars[st], d.bytes);
#pragma unroll
        for (int q = 0; q < PW; ++q)
            if (d.x[q] >= 0)
                tma_load_5d(dst + q * SLAB, &tmap, &bars[st], d.c0, d.z[q], d.y[q], d.x[q] + ii, d.m, policy);
    };

    const unsigned long long policy = l2_policy(a.evict_last);
    const int pp = lane / LPP;  // position within a group
    const int vl = lane % LPP;  // 16-byte lane vector within the CW chunk

    unsigned ph0 = 0, ph1 = 0;    // stage barrier parities
    unsigned rph0 = 0, rph1 = 0;  // record barrier parities
    GroupDesc<PW> d;

    fill(0);
    fill(1);
    if (!info[0].valid) return;
    mbar_wait(&rbar[0], rph0);
    rph0 ^= 1;
    if (lane == 0) {
        prepare(d, 0, 0);
        issue(d, 0, 0, policy);
    }
    int st = 0;  // stage of the step being consumed; the next step goes to st ^ 1

    int cslot = 0;
    while (true) {
        const ItemInfo it = info[cslot];
        const unsigned char *rc = recs + cslot * BP * RECB;
        for (int g = 0; g < it.G; ++g) {
            const int p = g * PW + pp;
            const T *w = reinterpret_cast<const T *>(rc + min(p, it.nb - 1) * RECB);
            T wx[12], wy[12], wz[12];
#pragma unroll
            for (int e = 0; e < 12; ++e) {
                wx[e] = w[e];
                wy[e] = w[12 + e];
                wz[e] = w[24 + e];
            }
            const int4 cell = *reinterpret_cast<const int4 *>(rc + min(p, it.nb - 1) * RECB + 36 * sizeof(T));
            AV acc[S][AN];
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
                for (int h = 0; h < AN; ++h) zero(acc[s][h]);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                // ---- issue the next step into the other stage (its previous
                // contents were consumed in the step before this one)
                __syncwarp();
                if (i < 3) {
                    if (lane == 0) issue(d, i + 1, st ^ 1, policy);
                } else if (g + 1 < it.G) {
                    if (lane == 0) {
                        prepare(d, cslot, g + 1);
                        issue(d, 0, st ^ 1, policy);
                    }
                } else if (info[cslot ^ 1].valid) {
                    // first group of the next item: its records must have landed
                    if (cslot) {
                        mbar_wait(&rbar[0], rph0);
                        rph0 ^= 1;
                    } else {
                        mbar_wait(&rbar[1], rph1);
                        rph1 ^= 1;
                    }
                    if (lane == 0) {
                        prepare(d, cslot ^ 1, 0);
                        issue(d, 0, st ^ 1, policy);
                    }
                }
                // ---- consume this step
                if (st) {
                    mbar_wait(&bars[1], ph1);
                    ph1 ^= 1;
                } else {
                    mbar_wait(&bars[0], ph0);
                    ph0 ^= 1;
                }
                const T *slab = reinterpret_cast<const T *>(ring + st * STAGE + pp * SLAB) + vl * W;
                slab_contract<KIND, CW>(slab, wy, wz, wx[i], wx[4 + i], wx[8 + i], acc);
                st ^= 1;
            }
            if constexpr (RATIO) {
                const bool live = p < it.nb;
                const long long gp = live ? cell.w : 0;
                const T *cf = reinterpret_cast<const T *>(a.coef) + gp * a.coef_stride + (long long)it.m * a.nb +
                              it.c * CW + vl * W;
                double part[S];
                ratio_partials<S, LPP>(acc, cf, live, part);  // reduced over the position's lanes
                if (live && vl == 0) {
                    const long long u = (long long)it.m * a.chunks + it.c;
                    double *dst = a.partials + (u * a.n_pos + gp) * S;
#pragma unroll
                    for (int s = 0; s < S; ++s) dst[s] = cell.x >= 0 ? part[s] : (double)NAN;
                }
            } else if (p < it.nb) {
                const long long gp = cell.w;  // original index
                const long long op = a.out_index ? a.out_index[gp] : gp;
                const long long lane = (long long)it.m * a.nb + it.c * CW + vl * W;
                T *o = reinterpret_cast<T *>(a.out) + op * a.out_pos_stride + lane;
                if (lane + W <= a.lane_limit)
                    store_lane<S>(o, a.out_stream_stride, acc, cell.x >= 0);
                else if (lane < a.lane_limit)
                    store_lane_partial<S>(o, a.out_stream_stride, acc, cell.x >= 0, (int)(a.lane_limit - lane));
            }
        }
        __syncwarp();
        const bool more = info[cslot ^ 1].valid;
        fill(cslot);  // the issue path has left this slot: refill it with the next ticket
        if (!more) break;
        cslot ^= 1;
    }
}

// ---------------------------------------------------------------- host --
typedef CUresult (*EncodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiled get_encode() {
    static EncodeTiled fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiled>(p);
    }
    return fn;
}

template <typename T>
constexpr size_t smem_bytes() {
    using C = typename TT<T>::Cfg;
    return (size_t)C::WARPS * C::R * STAGE + C::WARPS * (C::R + 2) * 8 + (size_t)C::WARPS * 2 * C::BP * TT<T>::RECB +
           C::WARPS * 2 * sizeof(ItemInfo);
}
static_assert(smem_bytes<float>() <= 232448, "shared memory budget");
static_assert(smem_bytes<double>() <= 232448, "shared memory budget");

template <int KIND, typename T, int CW, bool RATIO>
static int launch_t(const CUtensorMap &map, const Args &a, int sms, cudaStream_t st) {
    using C = typename TT<T>::Cfg;
    constexpr size_t sm = smem_bytes<T>();
    int grid = (int)min((long long)sms, (a.n_items + C::WARPS - 1) / C::WARPS);
    if (grid < 1) grid = 1;
    cudaFuncSetAttribute(eval_tma_kernel<KIND, T, CW, C, RATIO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sm);
    eval_tma_kernel<KIND, T, CW, C, RATIO><<<grid, C::WARPS * 32, sm, st>>>(map, a);
    return check_launch("spo_eval (tma) launch");
}

// chunk widths in elements: 128 / 256 / 512-byte rows (the fused ratio
// epilogue is instantiated for the 512-byte chunks only)
template <int KIND, typename T>
static int launch_cw(int cw_bytes, bool ratio, const CUtensorMap &map, const Args &a, int sms, cudaStream_t st) {
    constexpr int E = (int)sizeof(T);
    if (ratio) return launch_t<KIND, T, 512 / E, true>(map, a, sms, st);
    switch (cw_bytes) {
        case 128: return launch_t<KIND, T, 128 / E, false>(map, a, sms, st);
        case 256: return launch_t<KIND, T, 256 / E, false>(map, a, sms, st);
        default: return launch_t<KIND, T, 512 / E, false>(map, a, sms, st);
    }
}

template <typename T>
static int launch_kind(int kind, int cw_bytes, bool ratio, const CUtensorMap &map, const Args &a, int sms,
                       cudaStream_t st) {
    if (kind == SPO_KIND_V) return launch_cw<SPO_KIND_V, T>(cw_bytes, ratio, map, a, sms, st);
    if (kind == SPO_KIND_VGL) return launch_cw<SPO_KIND_VGL, T>(cw_bytes, ratio, map, a, sms, st);
    return launch_cw<SPO_KIND_VGH, T>(cw_bytes, ratio, map, a, sms, st);
}

// ratios[p][s] = sum over units u (in order) of partials[u][p][s]: deterministic.
__global__ void ratio_reduce_kernel(const double *__restrict__ partials, long long units, long long n,
                                    double *__restrict__ ratios) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (long long u = 0; u < units; ++u) s += partials[u * n + e];
        ratios[e] = s;
    }
}

constexpr long long ITEMS_PER_WARP_SMALL = 16, ITEMS_PER_WARP_FULL = 96;

static int rec_bytes(int dtype) { return dtype == SPO_F64 ? TT<double>::RECB : TT<float>::RECB; }
static int item_positions(int dtype) { return dtype == SPO_F64 ? TT<double>::Cfg::BP : TT<float>::Cfg::BP; }

}  // namespace tma

// workspace: [header: ticket | bucket counts | bucket cursors] [bucket id per
// position, 16-byte padded] [records, bucket-sorted]
long long eval_tma_workspace_bytes(int dtype, long long n_pos) {
    return tma::WS_HEADER + ((n_pos + 15) / 16) * 16 + n_pos * (long long)tma::rec_bytes(dtype);
}

// Extra workspace of the fused ratio epilogue: fp64 partials [units][n_pos][S]
// with units = n_tiles x (row bytes / 512); -1 when the row is not a multiple
// of 512 bytes (the epilogue runs with 512-byte chunks only).
long long eval_tma_ratio_bytes(int kind, int dtype, long long nb, long long n_tiles, long long n_pos) {
    const long long row = nb * (dtype == SPO_F64 ? 8 : 4);
    if (row % 512) return -1;
    const int S = kind == SPO_KIND_V ? 1 : (kind == SPO_KIND_VGL ? 5 : 10);
    return n_tiles * (row / 512) * n_pos * S * 8;
}

// Called by spo_eval for FAST requests with a workspace.  Returns -1 when the
// TMA path cannot be used (the caller then uses the generic kernel).
// cw_request: chunk width in elements (0 = automatic).  With `ratios` set the
// fused epilogue replaces the output stores: ratios[p][s] = sum_n
// stream_s(p, n) * coef[p][lane(n)] in fp64 (coef in output-lane layout).
int eval_tma(int kind, int dtype, const void *table, const TableGeom &geo, const GridArgs &g, const double *pos,
             long long n_pos, void *out, long long ops, long long oss, const long long *out_index, int *status,
             void *workspace, long long ws_bytes, cudaStream_t st, int cw_request, long long lane_limit,
             const void *coef = nullptr, long long coef_stride = 0, double *ratios = nullptr) {
    using namespace tma;
    const bool ratio = ratios != nullptr;
    const long long partial_bytes = ratio ? eval_tma_ratio_bytes(kind, dtype, geo.nb, geo.n_tiles, n_pos) : 0;
    if (ratio && partial_bytes < 0) return fail(SPO_ERR_CONFIG, "ratio epilogue needs rows of 512-byte multiples");
    if (!workspace || ws_bytes < eval_tma_workspace_bytes(dtype, n_pos) + partial_bytes || !aligned16(workspace))
        return ratio ? fail(SPO_ERR_CONTRACT, "workspace too small for the ratio epilogue") : -1;
    if (n_pos >= (1LL << 31)) return -1;  // records carry 32-bit original indices
    EncodeTiled encode = get_encode();
    if (!encode) return ratio ? fail(SPO_ERR_CUDA, "cuTensorMapEncodeTiled unavailable") : -1;
    if (ratio) cw_request = 512 / (dtype == SPO_F64 ? 8 : 4);
    const int E = dtype == SPO_F64 ? 8 : 4;
    // chunk width (bytes per row segment): one spatial block's rows x CW within
    // ~40 MB (a die's share of L2 with room for the next unit and the output
    // stream) -> 512 B for any realistic grid.
    const long long rows = (long long)geo.nxp * geo.nyp * geo.nzp;
    int cwb = cw_request * E;
    if (cwb == 0) {
        cwb = 128;
        if (rows * 512 / NBUCKET <= (40LL << 20)) cwb = 512;
        else if (rows * 256 / NBUCKET <= (40LL << 20)) cwb = 256;
    }
    while (cwb > 128 && (geo.nb * E) % cwb) cwb >>= 1;
    if (cwb != 128 && cwb != 256 && cwb != 512) return -1;
    if ((geo.nb * E) % cwb) return -1;
    const int cw = cwb / E;

    CUtensorMap map;
    cuuint64_t dims[5] = {(cuuint64_t)geo.nb, (cuuint64_t)geo.nzp, (cuuint64_t)geo.nyp, (cuuint64_t)geo.nxp,
                          (cuuint64_t)geo.n_tiles};
    cuuint64_t strides[4] = {(cuuint64_t)geo.nb * E, (cuuint64_t)geo.nzp * geo.nb * E,
                             (cuuint64_t)geo.nyp * geo.nzp * geo.nb * E, (cuuint64_t)geo.tile_stride * E};
    cuuint32_t box[5] = {(cuuint32_t)cw, 4, 4, 1, 1};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r = encode(&map, dtype == SPO_F64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                        5, const_cast<void *>(table), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(SPO_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long units = (long long)geo.n_tiles * (geo.nb / cw);
    const int BP = item_positions(dtype);
    const int pw = 32 * (16 / E) / cw;  // positions per warp step
    const long long warps = (long long)sms * (dtype == SPO_F64 ? TT<double>::Cfg::WARPS : TT<float>::Cfg::WARPS);
    // Item size: BP positions when every warp gets many items, fewer when it
    // gets few.  Measured (scripts/micro/item_size.py, interleaved medians):
    // smaller items cut the dynamic-scheduling tail and keep the in-flight
    // window inside fewer units (smaller L2 working set); at full size the
    // ticket and record traffic of small items costs more than that.
    const long long per_warp = units * ((n_pos + BP - 1) / BP) / warps;
    int bp = per_warp < ITEMS_PER_WARP_SMALL ? 2 : (per_warp < ITEMS_PER_WARP_FULL ? 4 : BP);
    bp = max(bp, pw);
    if (getenv("SPO_BP")) bp = max(1, min(BP, atoi(getenv("SPO_BP"))));
    if (((n_pos + bp - 1) / bp) * units >= (1LL << 32)) return -1;  // 32-bit tickets

    unsigned char *ws = static_cast<unsigned char *>(workspace);
    unsigned *counts = reinterpret_cast<unsigned *>(ws + 256);
    unsigned *cursors = reinterpret_cast<unsigned *>(ws + 512);
    unsigned char *bucket = ws + WS_HEADER;
    unsigned char *recs = ws + WS_HEADER + ((n_pos + 15) / 16) * 16;
    if (cudaMemsetAsync(ws, 0, WS_HEADER, st) != cudaSuccess) return check_launch("workspace reset");
    {
        long long blocks = (n_pos + 255) / 256;
        if (blocks > 148LL * 16) blocks = 148LL * 16;
        bucket_count_kernel<<<(unsigned)blocks, 256, 0, st>>>(g, pos, n_pos, bucket, counts);
        if (dtype == SPO_F64)
            prologue_records_kernel<double>
                <<<(unsigned)blocks, 256, 0, st>>>(g, pos, n_pos, bucket, counts, cursors, recs, status);
        else
            prologue_records_kernel<float>
                <<<(unsigned)blocks, 256, 0, st>>>(g, pos, n_pos, bucket, counts, cursors, recs, status);
        int rc = check_launch("spo_eval (prologue) launch");
        if (rc) return rc;
    }

    Args a;
    a.recs = recs;
    a.ticket = reinterpret_cast<unsigned *>(ws);
    a.n_pos = n_pos;
    a.bp = bp;
    a.nbatch = (n_pos + bp - 1) / bp;
    a.chunks = geo.nb / cw;
    a.n_items = a.nbatch * (long long)geo.n_tiles * a.chunks;
    a.nb = geo.nb;
    a.out = out;
    a.out_pos_stride = ops;
    a.out_stream_stride = oss;
    a.out_index = out_index;
    a.lane_limit = lane_limit;
    static const char *env_hint = getenv("SPO_L2HINT");
    a.evict_last = !(env_hint && env_hint[0] == '0');
    static const char *env_fence = getenv("SPO_PROXY_FENCE");
    a.proxy_fence = env_fence && env_fence[0] == '1';
    a.coef = coef;
    a.coef_stride = coef_stride;
    a.partials = ratio ? reinterpret_cast<double *>(ws + eval_tma_workspace_bytes(dtype, n_pos)) : nullptr;

    const int rc = dtype == SPO_F64 ? launch_kind<double>(kind, cwb, ratio, map, a, sms, st)
                                    : launch_kind<float>(kind, cwb, ratio, map, a, sms, st);
    if (rc || !ratio) return rc;
    const int S = kind == SPO_KIND_V ? 1 : (kind == SPO_KIND_VGL ? 5 : 10);
    const long long n = n_pos * S;
    const long long blocks = min((n + 255) / 256, 148LL * 16);
    ratio_reduce_kernel<<<(unsigned)blocks, 256, 0, st>>>(a.partials, (long long)geo.n_tiles * a.chunks, n, ratios);
    return check_launch("spo_eval_ratios (reduce) launch");
}

}  // namespace spo

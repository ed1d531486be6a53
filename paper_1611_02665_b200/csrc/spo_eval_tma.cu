// spo_eval_tma.cu -- TMA-pipelined fp32 V / VGL / VGH kernel (the fast path).
//
// Same math as spo_eval.cu's separable FAST contraction (kernels.py:143-247
// restated as k-, then j-, then i-sums with FMA), different data movement.
//
//  1. prologue_records_kernel: one thread per position maps it to (i0,j0,k0)
//     and the 36 fp32 basis weights, bit-exactly (spo_prologue.cuh), into a
//     160-byte record in the caller's workspace.  Once per position per call.
//  2. eval_tma_kernel: persistent CTAs (one per SM) of 8 warps.  Work items
//     are (unit u = (tile m, chunk c of CW lanes), batch of BP positions) and
//     are handed out by a global ticket counter in unit-major order, so at any
//     moment the whole GPU works on one or two units: the L2 working set is one
//     CW-wide slice of the table (rows x CW x 4 B, 38.5 MB for 67^3 at CW = 32)
//     -- the paper's AoSoA cache blocking, enforced by scheduling rather than by
//     hoping CTAs stay in step.
//     Per warp, a ring of R stages is fed by TMA: one cp.async.bulk.tensor.5d
//     per (position, i) brings the 4(j) x 4(k) x CW slab (16 rows) into shared
//     memory and completes on the stage's mbarrier; item records arrive by a
//     cp.async.bulk copy on their own mbarriers (double-buffered).  The warp
//     runs R-1 slabs ahead of its compute, across item boundaries.
//     Compute: lane = (position in group, 16-byte lane vector), 4 orbitals per
//     lane, S accumulators per orbital kept in registers over the 4 i-slabs,
//     streaming 16-byte stores.
#include <cuda.h>

#include <cstdlib>

#include "spo_common.cuh"
#include "spo_prologue.cuh"

namespace spo {
namespace tma {

constexpr int STAGE = 8192;   // bytes: 128 fp32 lanes x 16 rows
constexpr int REC = 40;       // floats per position record: 36 weights, i0, j0, k0, pad
constexpr int WS_HEADER = 1024;  // ticket @0, bucket counts @256, bucket cursors @512

struct Args {
    const float *recs;        // [n_pos][REC]
    unsigned *ticket;
    long long n_pos;
    long long nbatch;         // ceil(n_pos / BP)
    long long n_items;        // units * nbatch
    int chunks;               // chunks of CW lanes per tile row
    int nb;                   // table row length (lanes)
    float *out;
    long long out_pos_stride, out_stream_stride;
    const long long *out_index;
    int evict_last;           // L2 evict_last hint on table slabs
    int proxy_fence;          // fence.proxy.async before reusing a stage (diagnostic)
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

// Packed fp32x2 FMA (SASS FFMA2, sm_100): two independent round-to-nearest
// fp32 FMAs per instruction with a broadcast scalar multiplier -- bitwise the
// same as two __fmaf_rn, at half the issue slots.
__device__ __forceinline__ float2 fma2(float w, float2 c, float2 acc) {
    return __ffma2_rn(make_float2(w, w), c, acc);
}
__device__ __forceinline__ float2 mul2(float w, float2 c) { return __fmul2_rn(make_float2(w, w), c); }

// slab_fma with the 4 orbitals of a lane handled as two fp32x2 pairs.
template <int KIND, int CW>
__device__ __forceinline__ void slab_fma2(const float *__restrict__ slab, const float (&wy)[12],
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

// One i-slab of the separable contraction for one 16-byte lane vector.
// slab: [j][k][CW] floats of this lane's position; wy/wz: 12 weights each;
// ax/dax/d2ax: the x weights of this i.
template <int KIND, int CW>
__device__ __forceinline__ void slab_fma(const float *__restrict__ slab, const float (&wy)[12],
                                         const float (&wz)[12], float ax, float dax, float d2ax,
                                         float (&acc)[NS<KIND>::S][4]) {
    float t00[4], t10[4], t01[4], t20[4], t11[4], t02[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) t00[e] = t10[e] = t01[e] = t20[e] = t11[e] = t02[e] = 0.0f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        float4 c[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) c[k] = *reinterpret_cast<const float4 *>(slab + (j * 4 + k) * CW);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float c0 = (&c[0].x)[e], c1 = (&c[1].x)[e], c2 = (&c[2].x)[e], c3 = (&c[3].x)[e];
            const float s0 = __fmaf_rn(wz[3], c3, __fmaf_rn(wz[2], c2, __fmaf_rn(wz[1], c1, wz[0] * c0)));
            t00[e] = __fmaf_rn(wy[j], s0, t00[e]);
            if (KIND != SPO_KIND_V) {
                const float s1 = __fmaf_rn(wz[7], c3, __fmaf_rn(wz[6], c2, __fmaf_rn(wz[5], c1, wz[4] * c0)));
                const float s2 = __fmaf_rn(wz[11], c3, __fmaf_rn(wz[10], c2, __fmaf_rn(wz[9], c1, wz[8] * c0)));
                t10[e] = __fmaf_rn(wy[4 + j], s0, t10[e]);
                t01[e] = __fmaf_rn(wy[j], s1, t01[e]);
                t20[e] = __fmaf_rn(wy[8 + j], s0, t20[e]);
                t02[e] = __fmaf_rn(wy[j], s2, t02[e]);
                if (KIND == SPO_KIND_VGH) t11[e] = __fmaf_rn(wy[4 + j], s1, t11[e]);
            }
        }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        acc[0][e] = __fmaf_rn(ax, t00[e], acc[0][e]);
        if (KIND != SPO_KIND_V) {
            acc[1][e] = __fmaf_rn(dax, t00[e], acc[1][e]);
            acc[2][e] = __fmaf_rn(ax, t10[e], acc[2][e]);
            acc[3][e] = __fmaf_rn(ax, t01[e], acc[3][e]);
        }
        if (KIND == SPO_KIND_VGL)
            acc[4][e] = __fmaf_rn(d2ax, t00[e], __fmaf_rn(ax, t20[e], __fmaf_rn(ax, t02[e], acc[4][e])));
        if (KIND == SPO_KIND_VGH) {
            acc[4][e] = __fmaf_rn(d2ax, t00[e], acc[4][e]);
            acc[5][e] = __fmaf_rn(dax, t10[e], acc[5][e]);
            acc[6][e] = __fmaf_rn(dax, t01[e], acc[6][e]);
            acc[7][e] = __fmaf_rn(ax, t20[e], acc[7][e]);
            acc[8][e] = __fmaf_rn(ax, t11[e], acc[8][e]);
            acc[9][e] = __fmaf_rn(ax, t02[e], acc[9][e]);
        }
    }
}

// ------------------------------------------------------------ prologue --
// Positions are binned by the spatial block (NBK^3 blocks of the grid) of
// their stencil cell, so that the eval kernel's unit-major sweep touches one
// block's rows at a time: the L2 working set is (rows / NBK^3) x CW x 4 B,
// small enough for CW = 128 (one TMA per position-slab instead of four).
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

// pass 2: records (bit-exact mapping + 36 fp32 weights + cell + original
// index) scattered to their bucket's range; slots are reserved per block.
__global__ void prologue_records_kernel(GridArgs g, const double *__restrict__ pos, long long n,
                                        const unsigned char *__restrict__ bucket,
                                        const unsigned *__restrict__ counts, unsigned *__restrict__ cursors,
                                        float *__restrict__ recs, int *__restrict__ status) {
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
            float w[REC];
            weights_f32(tx, g.dinv[0], w);
            weights_f32(ty, g.dinv[1], w + 12);
            weights_f32(tz, g.dinv[2], w + 24);
            if (!(isfinite(x) && isfinite(y) && isfinite(z))) {
                if (status) atomicOr(status, 1);
                i0 = -1;
            }
            w[36] = __int_as_float(i0);
            w[37] = __int_as_float(j0);
            w[38] = __int_as_float(k0);
            w[39] = __int_as_float((int)p);  // original position index
            float4 *dst = reinterpret_cast<float4 *>(recs + (long long)(base[b] + rank) * REC);
#pragma unroll
            for (int e = 0; e < REC / 4; ++e) dst[e] = make_float4(w[4 * e], w[4 * e + 1], w[4 * e + 2], w[4 * e + 3]);
        }
        __syncthreads();
    }
}

// -------------------------------------------------------------- kernel --
// Launch shapes: warps per CTA, ring stages per warp, positions per item.
template <int WARPS_, int R_, int BP_>
struct TCfg {
    static constexpr int WARPS = WARPS_, R = R_, BP = BP_;
};
using CfgB = TCfg<12, 2, 8>;   // 12 warps, one slab in flight per warp while it computes one

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
    bool any;
};

template <int KIND, int CW, class C>
__global__ void __launch_bounds__(C::WARPS * 32, 1)
    eval_tma_kernel(const __grid_constant__ CUtensorMap tmap, const Args a) {
    constexpr int WARPS = C::WARPS, BP = C::BP;
    static_assert(C::R == 2, "the issue path runs exactly one slab ahead");
    constexpr int R = 2;
    constexpr int S = NS<KIND>::S;
    constexpr int PW = 128 / CW;       // positions per warp step
    constexpr int LPP = CW / 4;        // lanes per position
    constexpr int SLAB = CW * 16 * 4;  // bytes per (position, i) slab
    static_assert(PW * SLAB == STAGE, "stage must hold one warp step");
    static_assert(BP % PW == 0, "items hold whole groups");

    extern __shared__ __align__(1024) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char *ring = smem + (size_t)warp * R * STAGE;
    unsigned long long *bars =
        reinterpret_cast<unsigned long long *>(smem + (size_t)WARPS * R * STAGE) + warp * (R + 2);
    unsigned long long *rbar = bars + R;  // record barriers of slots 0/1
    float *recs = reinterpret_cast<float *>(smem + (size_t)WARPS * R * STAGE + WARPS * (R + 2) * 8) +
                  warp * 2 * BP * REC;
    ItemInfo *info = reinterpret_cast<ItemInfo *>(smem + (size_t)WARPS * R * STAGE + WARPS * (R + 2) * 8 +
                                                  WARPS * 2 * BP * REC * 4) + warp * 2;

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
                it.b0 = b * BP;
                it.nb = (int)min((long long)BP, a.n_pos - it.b0);
                it.G = (it.nb + PW - 1) / PW;
                if (a.proxy_fence) fence_proxy_async();  // WAR on the slot, see issue()
                mbar_arrive_expect_tx(&rbar[slot], (unsigned)(it.nb * REC * 4));
                bulk_load(recs + slot * BP * REC, a.recs + it.b0 * REC, (unsigned)(it.nb * REC * 4), &rbar[slot]);
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
        const float *rc = recs + slot * BP * REC;
        d.bytes = 0;
        d.c0 = it.c * CW;
        d.m = it.m;
#pragma unroll
        for (int q = 0; q < PW; ++q) {
            const int p = g * PW + q;
            const int4 cell = *reinterpret_cast<const int4 *>(rc + min(p, it.nb - 1) * REC + 36);
            const bool ok = p < it.nb && cell.x >= 0;
            d.x[q] = ok ? cell.x : -1;
            d.y[q] = cell.y;
            d.z[q] = cell.z;
            d.bytes += ok ? SLAB : 0;
        }
        d.any = true;
    };
    // lane 0: issue slab ii of the described group into stage st
    auto issue = [&](const GroupDesc<PW> &d, int ii, int st, unsigned long long policy) {
        unsigned char *dst = ring + st * STAGE;
        // WAR only (LDS reads of this stage, all consumed before the
        // __syncwarp above, then the TMA write): no proxy fence needed, as in
        // a consumer-release / producer-acquire TMA pipeline.
        if (a.proxy_fence) fence_proxy_async();
        mbar_arrive_expect_tx(&bars[st], d.bytes);
#pragma unroll
        for (int q = 0; q < PW; ++q)
            if (d.x[q] >= 0) tma_load_5d(dst + q * SLAB, &tmap, &bars[st], d.c0, d.z[q], d.y[q], d.x[q] + ii, d.m, policy);
    };

    const unsigned long long policy = l2_policy(a.evict_last);
    const int pp = lane / LPP;  // position within a group
    const int vl = lane % LPP;  // 16-byte lane vector within the CW chunk

    unsigned ph0 = 0, ph1 = 0;    // stage barrier parities
    unsigned rph0 = 0, rph1 = 0;  // record barrier parities
    GroupDesc<PW> d;
    d.any = false;

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
        const float *rc = recs + cslot * BP * REC;
        for (int g = 0; g < it.G; ++g) {
            const int p = g * PW + pp;
            const float *w = rc + min(p, it.nb - 1) * REC;
            float wx[12], wy[12], wz[12];
#pragma unroll
            for (int e = 0; e < 12; e += 4) {
                const float4 x4 = *reinterpret_cast<const float4 *>(w + e);
                const float4 y4 = *reinterpret_cast<const float4 *>(w + 12 + e);
                const float4 z4 = *reinterpret_cast<const float4 *>(w + 24 + e);
                wx[e] = x4.x, wx[e + 1] = x4.y, wx[e + 2] = x4.z, wx[e + 3] = x4.w;
                wy[e] = y4.x, wy[e + 1] = y4.y, wy[e + 2] = y4.z, wy[e + 3] = y4.w;
                wz[e] = z4.x, wz[e + 1] = z4.y, wz[e + 2] = z4.z, wz[e + 3] = z4.w;
            }
            const bool finite = __float_as_int(w[36]) >= 0;
            float2 acc[S][2];
#pragma unroll
            for (int s = 0; s < S; ++s) acc[s][0] = acc[s][1] = make_float2(0.0f, 0.0f);
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
                const float *slab = reinterpret_cast<const float *>(ring + st * STAGE + pp * SLAB) + vl * 4;
                slab_fma2<KIND, CW>(slab, wy, wz, wx[i], wx[4 + i], wx[8 + i], acc);
                st ^= 1;
            }
            if (p < it.nb) {
                const long long gp = __float_as_int(rc[p * REC + 39]);  // original index
                const long long op = a.out_index ? a.out_index[gp] : gp;
                float *o = a.out + op * a.out_pos_stride + (long long)it.m * a.nb + it.c * CW + vl * 4;
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const float4 v = finite ? make_float4(acc[s][0].x, acc[s][0].y, acc[s][1].x, acc[s][1].y)
                                            : make_float4(NAN, NAN, NAN, NAN);
                    __stcs(reinterpret_cast<float4 *>(o + s * a.out_stream_stride), v);
                }
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

template <class C>
constexpr size_t smem_bytes() {
    return (size_t)C::WARPS * C::R * STAGE + C::WARPS * (C::R + 2) * 8 + C::WARPS * 2 * C::BP * REC * 4 +
           C::WARPS * 2 * sizeof(ItemInfo);
}
static_assert(smem_bytes<CfgB>() <= 232448, "shared memory budget");

template <int KIND, int CW, class C>
static int launch_t(const CUtensorMap &map, const Args &a, int sms, cudaStream_t st) {
    constexpr size_t sm = smem_bytes<C>();
    const long long warps_needed = (a.n_items + 1) / 2;
    int grid = (int)min((long long)sms, (warps_needed + C::WARPS - 1) / C::WARPS);
    if (grid < 1) grid = 1;
    cudaFuncSetAttribute(eval_tma_kernel<KIND, CW, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    eval_tma_kernel<KIND, CW, C><<<grid, C::WARPS * 32, sm, st>>>(map, a);
    return check_launch("spo_eval (tma) launch");
}

template <int KIND, class C>
static int launch_cw(int cw, const CUtensorMap &map, const Args &a, int sms, cudaStream_t st) {
    switch (cw) {
        case 32: return launch_t<KIND, 32, C>(map, a, sms, st);
        case 64: return launch_t<KIND, 64, C>(map, a, sms, st);
        default: return launch_t<KIND, 128, C>(map, a, sms, st);
    }
}



}  // namespace tma

// workspace: [header: ticket | bucket counts | bucket cursors] [bucket id per
// position, 16-byte padded] [records, bucket-sorted]
long long eval_tma_workspace_bytes(long long n_pos) {
    return tma::WS_HEADER + ((n_pos + 15) / 16) * 16 + n_pos * tma::REC * 4;
}


// Called by spo_eval for fp32 FAST requests with a workspace.  Returns -1
// when the TMA path cannot be used (the caller then uses the generic kernel).
int eval_tma(int kind, const float *table, const TableGeom &geo, const GridArgs &g, const double *pos,
             long long n_pos, float *out, long long ops, long long oss, const long long *out_index, int *status,
             void *workspace, long long ws_bytes, cudaStream_t st, int cw_request) {
    using namespace tma;
    if (!workspace || ws_bytes < eval_tma_workspace_bytes(n_pos) || !aligned16(workspace)) return -1;
    EncodeTiled encode = get_encode();
    if (!encode) return -1;
    // chunk width: working set rows x CW x 4 B <= ~40 MB unless overridden (one
    // die's share of L2, with room for the next unit and the output stream)
    const long long rows = (long long)geo.nxp * geo.nyp * geo.nzp;
    int cw = cw_request;
    if (cw == 0) {
        cw = 32;
        if (rows * 128 * 4 / NBUCKET <= (40LL << 20)) cw = 128;
        else if (rows * 64 * 4 / NBUCKET <= (40LL << 20)) cw = 64;
    }
    while (cw > 32 && geo.nb % cw) cw >>= 1;
    if (cw < 32 || geo.nb % cw) return -1;

    CUtensorMap map;
    cuuint64_t dims[5] = {(cuuint64_t)geo.nb, (cuuint64_t)geo.nzp, (cuuint64_t)geo.nyp, (cuuint64_t)geo.nxp,
                          (cuuint64_t)geo.n_tiles};
    cuuint64_t strides[4] = {(cuuint64_t)geo.nb * 4, (cuuint64_t)geo.nzp * geo.nb * 4,
                             (cuuint64_t)geo.nyp * geo.nzp * geo.nb * 4, (cuuint64_t)geo.tile_stride * 4};
    cuuint32_t box[5] = {(cuuint32_t)cw, 4, 4, 1, 1};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float *>(table), dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(SPO_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);

    if (n_pos >= (1LL << 31)) return -1;  // records carry 32-bit original indices
    unsigned char *ws = static_cast<unsigned char *>(workspace);
    unsigned *counts = reinterpret_cast<unsigned *>(ws + 256);
    unsigned *cursors = reinterpret_cast<unsigned *>(ws + 512);
    unsigned char *bucket = ws + WS_HEADER;
    float *recs = reinterpret_cast<float *>(ws + WS_HEADER + ((n_pos + 15) / 16) * 16);
    if (cudaMemsetAsync(ws, 0, WS_HEADER, st) != cudaSuccess) return check_launch("workspace reset");
    {
        long long blocks = (n_pos + 255) / 256;
        if (blocks > 148LL * 16) blocks = 148LL * 16;
        bucket_count_kernel<<<(unsigned)blocks, 256, 0, st>>>(g, pos, n_pos, bucket, counts);
        prologue_records_kernel<<<(unsigned)blocks, 256, 0, st>>>(g, pos, n_pos, bucket, counts, cursors, recs,
                                                                  status);
        int rc = check_launch("spo_eval (prologue) launch");
        if (rc) return rc;
    }

    const int BP = CfgB::BP;
    Args a;
    a.recs = recs;
    a.ticket = reinterpret_cast<unsigned *>(ws);
    a.n_pos = n_pos;
    a.nbatch = (n_pos + BP - 1) / BP;
    a.chunks = geo.nb / cw;
    a.n_items = a.nbatch * (long long)geo.n_tiles * a.chunks;
    a.nb = geo.nb;
    a.out = out;
    a.out_pos_stride = ops;
    a.out_stream_stride = oss;
    a.out_index = out_index;
    static const char *env_hint = getenv("SPO_L2HINT");
    a.evict_last = !(env_hint && env_hint[0] == '0');
    static const char *env_fence = getenv("SPO_PROXY_FENCE");
    a.proxy_fence = env_fence && env_fence[0] == '1';
    if (a.n_items >= (1LL << 32)) return -1;  // 32-bit ticket counter

    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (kind == SPO_KIND_V) return launch_cw<SPO_KIND_V, CfgB>(cw, map, a, sms, st);
    if (kind == SPO_KIND_VGL) return launch_cw<SPO_KIND_VGL, CfgB>(cw, map, a, sms, st);
    return launch_cw<SPO_KIND_VGH, CfgB>(cw, map, a, sms, st);
}

}  // namespace spo

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
#include "spo_tma.cuh"

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
    int kmul;                   // k-power tables: cell k0's rows start at 4 k0
    double dz, dz2;             // k-power tables: 1/dz, 2/dz^2
};

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
                                        unsigned char *__restrict__ recs, int *__restrict__ status, int kpower) {
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
            if (kpower) w[24] = (T)tz;  // k-power tables: the z weight is t itself
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

template <int KIND, typename T, int CW, class C, bool RATIO, bool KP>
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
            d.z[q] = cell.z * a.kmul;
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
            T wx[12], wy[12], wz[12];
            load_weights(rc + min(p, it.nb - 1) * RECB, wx, wy, wz);
            const int4 cell = *reinterpret_cast<const int4 *>(rc + min(p, it.nb - 1) * RECB + 36 * sizeof(T));
            AV acc[S][AN], zs[4][AN];  // zs: fp32 z-second-derivative sums (slab_contract)
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
                for (int h = 0; h < AN; ++h) zero(acc[s][h]);
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int h = 0; h < AN; ++h) zero(zs[c][h]);
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
                if constexpr (KP) {
                    const T dz = (T)a.dz, dz2 = (T)a.dz2;
                    slab_contract_kp<KIND, CW>(slab, wy, wz[0], wx[i], wx[4 + i], wx[8 + i], mul_rn(wx[i], dz),
                                               mul_rn(wx[4 + i], dz), mul_rn(wx[i], dz2), acc);
                } else if constexpr (sizeof(T) == 4) {
                    slab_contract<KIND, CW>(slab, wy, wz, wx[i], wx[4 + i], wx[8 + i], acc, zs);
                } else {
                    slab_contract<KIND, CW>(slab, wy, wz, wx[i], wx[4 + i], wx[8 + i], acc);
                }
                st ^= 1;
            }
            if constexpr (!KP && sizeof(T) == 4) finish_z2<KIND>(wz, zs, acc);
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
template <typename T>
constexpr size_t smem_bytes() {
    using C = typename TT<T>::Cfg;
    return (size_t)C::WARPS * C::R * STAGE + C::WARPS * (C::R + 2) * 8 + (size_t)C::WARPS * 2 * C::BP * TT<T>::RECB +
           C::WARPS * 2 * sizeof(ItemInfo);
}
static_assert(smem_bytes<float>() <= 232448, "shared memory budget");
static_assert(smem_bytes<double>() <= 232448, "shared memory budget");

template <int KIND, typename T, int CW, bool RATIO, bool KP = false>
static int launch_t(const CUtensorMap &map, const Args &a, int sms, cudaStream_t st) {
    using C = typename TT<T>::Cfg;
    constexpr size_t sm = smem_bytes<T>();
    int grid = (int)min((long long)sms, (a.n_items + C::WARPS - 1) / C::WARPS);
    if (grid < 1) grid = 1;
    cudaFuncSetAttribute(eval_tma_kernel<KIND, T, CW, C, RATIO, KP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sm);
    eval_tma_kernel<KIND, T, CW, C, RATIO, KP><<<grid, C::WARPS * 32, sm, st>>>(map, a);
    return check_launch("spo_eval (tma) launch");
}

// chunk widths in elements: 128 / 256 / 512-byte rows (the fused ratio
// epilogue is instantiated for the 512-byte chunks only)
template <int KIND, typename T>
static int launch_cw(int cw_bytes, bool ratio, const CUtensorMap &map, const Args &a, int sms, cudaStream_t st) {
    constexpr int E = (int)sizeof(T);
    if (ratio) return launch_t<KIND, T, 512 / E, true>(map, a, sms, st);
    if (a.kmul != 1) {  // k-power tables (the ratio epilogue takes B-spline tables only)
        switch (cw_bytes) {
            case 128: return launch_t<KIND, T, 128 / E, false, true>(map, a, sms, st);
            case 256: return launch_t<KIND, T, 256 / E, false, true>(map, a, sms, st);
            default: return launch_t<KIND, T, 512 / E, false, true>(map, a, sms, st);
        }
    }
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

int ratio_reduce(int kind, const double *partials, long long units, long long n_pos, double *ratios,
                 cudaStream_t st);

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
    if (!tensor_map_encoder()) return ratio ? fail(SPO_ERR_CUDA, "cuTensorMapEncodeTiled unavailable") : -1;
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
    const int r = table_tensor_map(&map, table, geo, dtype, cw);
    if (r) return fail(SPO_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", r);
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
        const Grid1D pg = prologue_grid(n_pos);
        bucket_count_kernel<<<pg.blocks, pg.threads, 0, st>>>(g, pos, n_pos, bucket, counts);
        if (dtype == SPO_F64)
            prologue_records_kernel<double>
                <<<pg.blocks, pg.threads, 0, st>>>(g, pos, n_pos, bucket, counts, cursors, recs, status,
                                                   geo.kmul != 1);
        else
            prologue_records_kernel<float>
                <<<pg.blocks, pg.threads, 0, st>>>(g, pos, n_pos, bucket, counts, cursors, recs, status,
                                                   geo.kmul != 1);
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
    a.kmul = geo.kmul;
    a.dz = g.dinv[2];
    a.dz2 = 2.0 * g.dinv[2] * g.dinv[2];
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
    return ratio_reduce(kind, a.partials, (long long)geo.n_tiles * a.chunks, n_pos, ratios, st);
}

// ratios[p][s] = sum over the units of partials[u][p][s] (fixed order)
int ratio_reduce(int kind, const double *partials, long long units, long long n_pos, double *ratios,
                 cudaStream_t st) {
    const int S = kind == SPO_KIND_V ? 1 : (kind == SPO_KIND_VGL ? 5 : 10);
    const long long n = n_pos * S;
    const long long blocks = min((n + 255) / 256, 148LL * 16);
    tma::ratio_reduce_kernel<<<(unsigned)blocks, 256, 0, st>>>(partials, units, n, ratios);
    return check_launch("spo_eval_ratios (reduce) launch");
}

}  // namespace spo
